"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see looptile_oracle.py)."""
