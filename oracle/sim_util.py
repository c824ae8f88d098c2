"""The reference simulator's SIMT utilisation for the configurations of the
ncu lane-efficiency sweep (tools/lane_eff_driver.py), so the two can be read
side by side.  TEST / MEASUREMENT INFRASTRUCTURE (runs the reference itself,
oracle/_ref).  With every latency 1 (LatencyModel::fromFile, ir.cpp:246-280)
usefulThreadCycles / threadCycles is the interpreter's counterpart of ncu's
thread_inst_executed / (32 x inst_executed).

    python oracle/sim_util.py > profiles/r01_simulator_util.json
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle import Reference  # noqa: E402

CORPUS = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested", "bitonic"]
UNIT = [1] * 28


def util(mod, warp, n_warps, seed, override):
    prog_g = sum(s for _, s in mod.globals)
    prog_s = sum(s for _, s in mod.shared)
    args = np.zeros((len(mod.params), n_warps), np.int32)
    gl = np.zeros((n_warps, prog_g), np.int32)
    sh = np.zeros((n_warps, max(1, prog_s)), np.int32)
    for w in range(n_warps):
        a, g, s = mod.make_random_input(warp, seed + w)
        args[:, w] = a
        gl[w] = g[:prog_g]
        sh[w, :prog_s] = s[:prog_s]
    for i, v in override.items():
        args[i, :] = v
    _, _, _, st = mod.execute_program(warp, n_warps, args, gl, sh[:, :prog_s].copy() if prog_s else None,
                                      latency=UNIT, threads=os.cpu_count() or 1)
    return float(st[:, 2].sum() / st[:, 1].sum())


def main():
    ref = Reference()
    out = {}
    for k in CORPUS:
        row = {}
        for tag, meld in (("unmelded", 0), ("melded", 1)):
            mod = ref.load(k, meld)
            ov = {} if k == "bitonic" else ({0: 16} if len(mod.params) == 1 else {0: 16, 1: 24})
            row[tag] = util(mod, 32, 2048, 1000, ov)
        out[k if k != "bitonic" else "bitonic_step"] = row
    print(json.dumps({"what": "reference simulator, unit latencies, warp 32, 2048 makeRandomInput warps, "
                              "half-warp split (n = 16; h = 16, q = 24)", "utilization": out}, indent=1))


if __name__ == "__main__":
    main()
