"""Condense an `ncu --page raw --csv` export (one kernel) into the JSON summary
committed under profiles/: duration, DRAM bytes, tensor-pipe and SM activity,
the top warp-stall reasons. Usage: python profiles/ncu_summary.py raw.csv out.json"""
import csv
import json
import sys

KEYS = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "sm__cycles_elapsed.avg",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "launch__shared_mem_per_block_dynamic", "launch__registers_per_thread",
]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(vals, units)))
    out = {k: {"value": d[k][0], "unit": d[k][1]} for k in KEYS if k in d}
    stalls = sorted(((float(v[0].replace(",", "") or 0), k) for k, v in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                    reverse=True)[:6]
    out["top_stall_samples"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): v for v, k in stalls}
    json.dump(out, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
