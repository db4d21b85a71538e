"""Summarise ncu --set full reports (gpurun_out/*.ncu-rep) into one JSON:
python scripts/ncu_summary.py out.json rep1.ncu-rep [rep2 ...]"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size"]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: r[i] for i, h in enumerate(hdr)}
        u = {h: units[i] for i, h in enumerate(hdr)}
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                item[k] = f"{d[k]} {u[k]}".strip()
        stalls = []
        for h, v in d.items():
            if "smsp__average_warps_issue_stalled" in h and "per_issue_active" in h:
                try:
                    stalls.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "")
                                   .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        item["top_stalls_per_issue"] = {h: round(v, 3) for v, h in sorted(stalls, reverse=True)[:4]}
        res.append(item)
    return res


if __name__ == "__main__":
    out = {rep.split("/")[-1]: summarise(rep) for rep in sys.argv[2:]}
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1)[:6000])
