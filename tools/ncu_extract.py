"""Condense an ncu report on the GPU box (reports are ~23 MB each; gpurun merges at most
64 MiB back): selected raw metrics -> <out>_details.csv, source page aggregated by CUDA
source line (instructions, shared-memory wavefronts, stall samples) -> <out>_source.txt.
usage: python tools/ncu_extract.py report.ncu-rep out_prefix"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ['Kernel Name', 'Block Size', 'Grid Size', 'gpu__time_duration.sum', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed.avg.per_cycle_elapsed',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__sass_inst_executed_op_shared_ld.sum',
        'smsp__sass_inst_executed_op_shared_st.sum', 'smsp__sass_inst_executed_op_global_ld.sum',
        'smsp__sass_inst_executed_op_global_st.sum', 'smsp__inst_executed_op_ldgsts.sum',
        'smsp__sass_inst_executed_op_tma_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread',
        'launch__shared_mem_per_block_dynamic', 'launch__occupancy_limit_shared_mem',
        'launch__occupancy_limit_registers', 'smsp__thread_inst_executed_per_inst_executed.ratio']
lines = ['metric,unit,value']
for w in want:
    if w in hdr:
        i = hdr.index(w)
        lines.append(f'"{w}","{units[i]}","{vals[i]}"')
for i, h in enumerate(hdr):
    if 'issue_stalled' in h and h.endswith('per_warp_active.pct'):
        lines.append(f'"{h}","{units[i]}","{vals[i]}"')
open(out + "_details.csv", "w").write("\n".join(lines) + "\n")

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
names = ("Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
         "# Samples")
agg, text = defaultdict(lambda: defaultdict(float)), {}
fname = h = None
for r in csv.reader(src.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        h = r
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    k = (fname, ln)
    text[k] = r[1][:80]
    for n in names:
        try:
            agg[k][n] += float(r[h.index(n)])
        except (ValueError, IndexError):
            pass
tot = {n: sum(a[n] for a in agg.values()) or 1.0 for n in names}
o = [str(tot)]
for n in ("L1 Wavefronts Shared", "Instructions Executed", "# Samples"):
    o.append("--- by " + n)
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][n])[:25]:
        o.append(f"{100*a['L1 Wavefronts Shared']/tot['L1 Wavefronts Shared']:5.1f}%wf "
                 f"inst {100*a['Instructions Executed']/tot['Instructions Executed']:4.1f}%  "
                 f"smp {100*a['# Samples']/tot['# Samples']:4.1f}%  {k[0]}:{k[1]}  {text[k]}")
open(out + "_source.txt", "w").write("\n".join(o) + "\n")
print(open(out + "_details.csv").read())
