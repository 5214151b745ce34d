"""Per-phase cycle accounting of the dataflow executor (profiling build:
`make -C paper_1708_03183_b200/csrc timing` -> libltcuda_timing.so, -DLT_PHASE_TIMING).
usage: LT_LIB_PATH=.../libltcuda_timing.so python tools/phase_timing.py CONFIG [ts] [nx ny]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1708_03183_b200 as lt
from paper_1708_03183_b200 import _lib
from paper_1708_03183_b200 import workloads as W
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
over = {}
if len(sys.argv) > 2: over["ts"] = int(sys.argv[2])
if len(sys.argv) > 4: over.update(nx=int(sys.argv[3]), ny=int(sys.argv[4]))
w = W.workload(cfgn, **over)
pb = W.build_problem(w)
sched = lt.inspect_chain(pb.chain, w.ts, lt.ExecMode.SHARED)
r = W.tiled_runner(pb, sched, repeats=w.chains_per_step)
lib = _lib.load()
buf = (C.c_ulonglong * 64)()
for _ in range(2): r()
torch.cuda.synchronize()
lib.lt_phase_cycles(buf, 1)
n = 3
for _ in range(n): r()
torch.cuda.synchronize()
lib.lt_phase_cycles(buf, 1)
cnt = buf[5]
names = {0: "blob wait", 1: "gather RW + wait", 2: "store-back", 3: "dep wait", 4: "tile total (after wait)"}
print(f"config {cfgn} {w.nx}x{w.ny} P{w.p} T{w.T} ts {w.ts}: executor {r.executor} wide {r.wide_build} "
      f"smem {r.smem_bytes}; tile instances {cnt}  (cycles per tile instance, thread 0)")
for k, v in names.items(): print(f"  {v:26s} {buf[k]/cnt:9.0f}")
for j in range(24):
    if buf[8 + j]: print(f"  loop {j:2d} total            {buf[8+j]/cnt:9.0f}" + (f"   records {buf[40+j]/cnt:7.0f}" if buf[40+j] else ""))
