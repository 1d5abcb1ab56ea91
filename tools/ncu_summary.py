"""Print the key counters of an ncu report (run here, no GPU needed)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__sass_inst_executed_op_shared_ld.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__warps_eligible.avg.per_cycle_active',
        'smsp__warps_active.avg.per_cycle_active', 'launch__registers_per_thread',
        'sm__cycles_elapsed.avg', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'lts__t_sectors_srcunit_tex_op_read.sum']
for vals in rows[2:]:
    print("----")
    d = dict(zip(hdr, vals))
    for w in want:
        if w in d:
            print(f"{w:70s} {d[w]}")
    try:
        cyc = float(d['sm__cycles_elapsed.avg'])
        wf = float(d['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'])
        print(f"{'smem wavefront utilisation (wavefronts / (148*cycles))':70s} {wf / (148 * cyc):.3f}")
    except (KeyError, ValueError):
        pass
    st = []
    for h, v in d.items():
        if 'warps_issue_stalled' in h and h.endswith('per_issue_active.ratio'):
            try:
                st.append((float(v), h.replace('smsp__average_warps_issue_stalled_', '')))
            except ValueError:
                pass
    for v, h in sorted(st, reverse=True)[:7]:
        print(f"   stall {v:7.3f} {h}")
