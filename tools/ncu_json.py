"""Summarise one kernel of an ncu --set full report as JSON (unit-aware).

    python tools/ncu_json.py <report.ncu-rep> <out.json> <workload name>

bench.py reads `dram_bytes_per_launch` of profiles/r02/ncu_quad_cfg{c}.json as roofline.traffic.
"""
import csv, json, subprocess, sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6, "%": 1}
rep, out, workload = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
d = {k: float(x.replace(",", "")) * SCALE.get(un, 1) for k, un, x in zip(h, u, v) if x.replace(",", "").replace(".", "", 1).isdigit()}
cyc = d["sm__cycles_elapsed.avg"]
res = {
    "kernel": [x for k, x in zip(h, v) if k == "Kernel Name"][0],
    "workload": workload,
    "capture": "ncu --set full --clock-control none --import-source on -s 1 -c 1 (tools/gpu_round.sh)",
    "gpu_time_ms": d["gpu__time_duration.sum"],
    "dram_read_bytes": d["dram__bytes_read.sum"],
    "dram_write_bytes": d["dram__bytes_write.sum"],
    "dram_bytes_per_launch": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
    "fp64_pipe_pct_of_peak": d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
    "smem_wavefront_utilisation": round(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"] / (148 * cyc), 3),
    "issue_active_pct": d["smsp__issue_active.avg.pct_of_peak_sustained_active"],
    "registers_per_thread": d["launch__registers_per_thread"],
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
