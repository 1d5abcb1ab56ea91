"""Hot-spot summary of an ncu report's SASS page: python tools/ncu_hot.py REPORT.ncu-rep [KERNEL_REGEX]
Prints headline metrics and the SASS regions (runs of equal execution count) with their
share of executed instructions and of stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2] if len(rows) > 2 else rows[1]
want = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts.sum"]
d = dict(zip(hdr, vals))
for k in want:
    if k in d:
        print(f"{k:70s} {d[k]}")
if "l1tex__data_pipe_lsu_wavefronts.sum" in d:
    wf = float(d["l1tex__data_pipe_lsu_wavefronts.sum"].replace(",", ""))
    cyc = float(d["sm__cycles_elapsed.avg"].replace(",", ""))
    print(f"{'LSU data-pipe utilisation (wavefronts / (148 cycles))':70s} {wf / (148 * cyc):.3f}")
for k, v in d.items():
    if "issue_stalled" in k and k.endswith("per_issue_active.ratio") and float(v or 0) > 0.15:
        print(f"   stall {float(v):6.3f} {k.split('issue_stalled_')[1]}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr, data = rows[1], rows[2:]
isrc, iex, ismp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("# Samples")
tot = sum(int(r[iex]) for r in data)
tots = sum(int(r[ismp]) for r in data)
print("total warp instructions", tot, "samples", tots)
blocks, cur = [], None
for k, r in enumerate(data):
    e, s = int(r[iex]), int(r[ismp])
    if cur and abs(e - cur["e"]) <= 0.02 * max(e, cur["e"], 1):
        cur["n"] += 1; cur["s"] += s; cur["end"] = k; cur["tot"] += e
    else:
        cur = {"e": e, "n": 1, "s": s, "start": k, "end": k, "tot": e}
        blocks.append(cur)
for b in blocks:
    if b["tot"] > 0.01 * tot or b["s"] > 0.01 * tots:
        print(f"sass[{b['start']:4d}-{b['end']:4d}] n={b['n']:4d} exec/inst={b['e']:.3e} "
              f"inst%={100 * b['tot'] / tot:5.1f} samples%={100 * b['s'] / tots:5.1f}")
if len(sys.argv) > 2:
    lo, hi = [int(v) for v in sys.argv[2].split("-")]
    for k in range(lo, hi + 1):
        print(k, data[k][isrc][:100], data[k][ismp])
