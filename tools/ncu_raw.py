"""Print selected raw ncu metrics (from `ncu --page raw --csv` dumps) side by side for several captures."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__m_l1tex2xbar_write_sectors_mem_lg_op_st.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg", "sm__cycles_active.avg"]


def load(p):
    rows = list(csv.reader(open(p)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


if __name__ == "__main__":
    ds = [load(p) for p in sys.argv[1:]]
    extra = [k for k in ds[0][0] if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    for k in KEYS + extra:
        vals = [d.get(k, "-") for d, _ in ds]
        if extra and k in extra:
            try:
                if max(float(v) for v in vals) < 0.3:
                    continue
            except ValueError:
                continue
            name = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
        else:
            name = k
        print(f"{name:75s} " + " ".join(f"{v:>14s}" for v in vals))
