"""Compact per-kernel summary of an ncu report (run here, on the CPU box):
    python tools/summarize_ncu.py gpurun_out/prof.ncu-rep > profiles/rNN_xxx.json
Keeps duration, DRAM bytes, throughput percentages, issue/occupancy, pipe utilisation, DFMA counts
and the warp-stall breakdown -- the numbers DESIGN.md and bench.py cite."""
import csv
import io
import json
import subprocess
import sys

RAW_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "derived__sm__sass_thread_inst_executed_op_dfma_pred_on_x2", "sm__ops_path_tensor_src_fp64.sum",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
             "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")[:120], "units": "bytes for dram__*, ms for gpu__time_duration"}
        for key in RAW_KEYS:
            if key in d:
                try:
                    v = float(d[key].replace(",", ""))
                    u = units.get(key, "")
                    if key.startswith("dram__bytes") or key == "gpu__time_duration.sum":
                        v *= scale.get(u, 1.0)
                    k[key] = v
                except ValueError:
                    k[key] = d[key]
        stalls = {c.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(d[c] or 0)
                  for c in hdr if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued")}
        tot = sum(stalls.values()) or 1.0
        k["stall_share"] = {s: round(v / tot, 4) for s, v in sorted(stalls.items(), key=lambda x: -x[1]) if v / tot > 0.01}
        out.append(k)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
