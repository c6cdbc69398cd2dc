"""Summarise an ncu --set full report (raw page) into the metrics we track."""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__waves_per_multiprocessor",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__sass_branch_targets_threads_divergent.sum",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__sass_inst_executed_op_global_ld.sum",
    "smsp__sass_inst_executed_op_global_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for name in WANT:
            if name in hdr:
                i = hdr.index(name)
                d[name] = f"{r[i]} {units[i]}".strip()
        # stall reasons (top)
        st = []
        for i, name in enumerate(hdr):
            if name.startswith("smsp__average_warp_latency_issue_stalled_") and name.endswith(".ratio"):
                try:
                    st.append((float(r[i]), name.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", "")))
                except ValueError:
                    pass
        if not st:
            for i, name in enumerate(hdr):
                if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
                    try:
                        st.append((float(r[i]), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
        st.sort(reverse=True)
        d["top_stalls"] = st[:6]
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps(summarise(p), indent=1))
