"""Summarise an ncu raw CSV export (one kernel launch): throughput, pipes, stalls."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    vals = rows[2] if len(rows) > 2 else rows[1]
    return dict(zip(hdr, vals))


def fl(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return float("nan")


KEYS = [
    ("duration_us", "gpu__time_duration.sum"),
    ("sm_clock_ghz", "smsp__cycles_elapsed.avg.per_second"),
    ("dram_read_bytes", "dram__bytes_read.sum"),
    ("dram_write_bytes", "dram__bytes_write.sum"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("smem_pct_peak", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("ipc", "sm__inst_executed.avg.per_cycle_active"),
    ("warps_active", "sm__warps_active.avg.per_cycle_active"),
    ("regs", "launch__registers_per_thread"),
    ("block", "launch__block_size"),
    ("grid", "launch__grid_size"),
    ("local_ld", "smsp__sass_inst_executed_op_local_ld.sum"),
    ("local_st", "smsp__sass_inst_executed_op_local_st.sum"),
    ("inst_executed", "smsp__inst_executed.sum"),
]


def main():
    for path in sys.argv[1:]:
        d = load(path)
        print(f"== {path}")
        for name, key in KEYS:
            if key in d:
                print(f"  {name:18s} {d[key]:>16s}  ({key})")
        st = [(k, fl(v)) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        st.sort(key=lambda kv: -kv[1])
        print("  stalls per issued instruction:")
        for k, v in st[:9]:
            print(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:24s} {v:.3f}")


if __name__ == "__main__":
    main()
