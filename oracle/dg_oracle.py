"""Elastic-wave DG kernels for the CPU oracle -- TEST INFRASTRUCTURE ONLY (stub)."""


def kernel_table():
    return {}
