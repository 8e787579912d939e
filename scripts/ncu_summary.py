"""Summarise an ncu --set full report (key throughput / memory / stall metrics)."""
import csv, io, subprocess, sys, json

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum",
        "smsp__average_warp_latency_issue_stalled_short_scoreboard",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum"]


def main(path, kernel=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if kernel and kernel not in d.get("Kernel Name", ""):
            continue
        item = {"kernel": d.get("Kernel Name", "")[:60]}
        for k in KEYS:
            if k in d:
                item[k] = d[k]
        stalls = {h: d[h] for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled")
                  or h.startswith("smsp__pcsamp_warps_issue_stalled")}
        top = sorted(((float(v.replace(",", "")), h) for h, v in stalls.items()
                      if v.replace(",", "").replace(".", "").isdigit()), reverse=True)[:8]
        item["top_stalls"] = [(h.split("stalled_")[-1], v) for v, h in top]
        res.append(item)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
