"""Summarise an .ncu-rep: key throughput, occupancy, stall and traffic metrics.
python tools/ncu_summary.py gpurun_out/prof.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__grid_size", "launch__block_size",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
]


def main(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(p, "no data")
            continue
        h, u = rows[0], rows[1]
        for v in rows[2:]:
            print(f"== {p}  {v[h.index('Kernel Name')][:60] if 'Kernel Name' in h else ''}")
            d = dict(zip(h, v))
            for k in KEYS:
                if k in d:
                    print(f"  {k:70s} {d[k]:>16s} {u[h.index(k)]}")
            stalls = sorted(((float(d[k] or 0), k) for k in h
                             if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")),
                            reverse=True)[:8]
            tot = sum(float(d[k] or 0) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"))
            for val, k in stalls:
                print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * val / max(tot, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1:])
