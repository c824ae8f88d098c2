"""Summarise an .ncu-rep (ncu --set full) into the metrics the judge and DESIGN.md cite.

    python tools/ncu_summary.py gpurun_out/prof_bitonic.ncu-rep > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "thread_inst_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    "thread_inst_pred_on_per_inst": ("smsp__thread_inst_executed_pred_on_per_inst_executed.ratio", 1),
    "branch_uniform_pct": ("smsp__sass_average_branch_targets_threads_uniform.pct", 1),
    "warp_inst_executed": ("smsp__inst_executed.sum", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    "sm_clock_hz": ("smsp__cycles_elapsed.avg.per_second", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e3, "ns": 1, "ms": 1e6,
              "usecond": 1e3, "nsecond": 1, "msecond": 1e6}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")]}
        for key, (metric, _) in METRICS.items():
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if key.startswith("dram_") and key.endswith("bytes"):
                v *= UNIT_SCALE.get(u, 1)
            if key == "duration_us":
                v = v * UNIT_SCALE.get(u, 1) / 1e3
            k[key] = v
        # warp-state breakdown: cycles stalled per issued instruction, by reason
        stalls = {}
        for i, h in enumerate(hdr):
            m = h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
            if m:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        if stalls:
            k["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        if "thread_inst_per_inst" in k:
            k["lane_efficiency"] = k["thread_inst_per_inst"] / 32.0
        if "thread_inst_pred_on_per_inst" in k:
            k["lane_efficiency_pred_on"] = k["thread_inst_pred_on_per_inst"] / 32.0
        if "dram_read_bytes" in k and "dram_write_bytes" in k:
            k["dram_bytes"] = k["dram_read_bytes"] + k["dram_write_bytes"]
        kernels.append(k)
    return kernels


if __name__ == "__main__":
    print(json.dumps({"source": sys.argv[1], "kernels": summarise(sys.argv[1])}, indent=1))
