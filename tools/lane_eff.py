"""Summarise an ncu metrics CSV of tools/lane_eff_driver.py into per-kernel,
per-form SIMT lane efficiency (instruction-weighted over the kernel's launches):
    thread_inst / (32 * inst)          smsp__thread_inst_executed_per_inst_executed
    pred_on thread_inst / (32 * inst)  ..._pred_on_per_inst_executed
    branch uniformity                  smsp__sass_average_branch_targets_threads_uniform.pct
"""
import csv
import json
import re
import sys
from collections import defaultdict

M_TI = "smsp__thread_inst_executed_per_inst_executed.ratio"
M_TP = "smsp__thread_inst_executed_pred_on_per_inst_executed.ratio"
M_BU = "smsp__sass_average_branch_targets_threads_uniform.pct"
M_IN = "smsp__inst_executed.sum"
M_T = "gpu__time_duration.sum"


def label(name):
    """(family, form) from a demangled kernel name, or None for kernels not ours."""
    base = re.sub(r"^void\s+", "", name).split("(")[0]
    base = base.replace("darm_gpu::", "")
    fam, _, targs = base.partition("<")
    args = [a.strip() for a in targs.rstrip(">").split(",")] if targs else []
    def form(x):
        return {"1": "melded", "true": "melded", "2": "predicated", "3": "melded_literal"}.get(x, "unmelded")
    if fam == "corpus_lanes":
        k = args[0].lower()
        k = {"sb2t<0>": "sb2", "sb2t<1>": "sb2r", "sb3t<0>": "sb3", "sb3t<1>": "sb3r", "sb4t<0>": "sb4",
             "sb4t<1>": "sb4r", "sb2t<false>": "sb2", "sb2t<true>": "sb2r", "sb3t<false>": "sb3",
             "sb3t<true>": "sb3r", "sb4t<false>": "sb4", "sb4t<true>": "sb4r"}.get(k, k)
        return k, form(args[1])
    if fam == "bitonic_step_kernel":
        return "bitonic_step", form(args[0])
    if fam == "bitonic_sort_reg_kernel":
        return f"bitonic_sort_{args[2]}kpt", form(args[0])
    if fam == "bitonic_sort_kernel":
        return "bitonic_sort_1kpt", form(args[0])
    if fam == "oddeven_sort_reg_kernel":
        return f"pcm_{args[2]}kpt", form(args[0])
    if fam == "oddeven_sort_kernel":
        return "pcm_1kpt", form(args[0])
    if fam in ("merge_sort_tile_kernel", "merge_sort_pass_kernel"):
        return "ms", form(args[0])
    if fam == "nqueens_kernel":
        return "nqueens", form(args[0])
    if fam == "nqueens_step_kernel":
        return "nqueens_paper_shape", form(args[0])
    if fam == "lud_panel_kernel":
        return "lud_panel", form(args[0])
    if fam == "srad_sweep_kernel":
        return ("srad_fast" if args[1] in ("1", "true") else "srad"), form(args[0])
    return None


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    idi = h.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        names[r[idi]] = r[ki]
    acc = defaultdict(lambda: defaultdict(float))
    for lid, m in per.items():
        lab = label(names[lid])
        if lab is None or M_IN not in m:
            continue
        a = acc[lab]
        a["inst"] += m[M_IN]
        a["thread"] += m.get(M_TI, 0) * m[M_IN]
        a["pred"] += m.get(M_TP, 0) * m[M_IN]
        a["bu"] += m.get(M_BU, 0) * m[M_IN]
        a["launches"] += 1
    out = defaultdict(dict)
    for (fam, form), a in sorted(acc.items()):
        out[fam][form] = {"lane_efficiency": a["thread"] / a["inst"] / 32, "lane_efficiency_pred_on":
                          a["pred"] / a["inst"] / 32, "branch_uniform_pct": a["bu"] / a["inst"],
                          "warp_inst": a["inst"], "launches": int(a["launches"])}
    return out


if __name__ == "__main__":
    print(json.dumps({"source": sys.argv[1], "kernels": summarise(sys.argv[1])}, indent=1))
