"""Markdown tables for DESIGN.md §8 from the committed profiles:
bench per-kernel rows (profiles/rNN_bench.json) and the ncu lane-efficiency
sweep (profiles/rNN_lane_efficiency.json, the latest *_simulator_util.json).

    python tools/design_tables.py [rNN]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def t(us):
    return f"{us / 1e3:.2f} ms" if us >= 1000 else f"{us:.1f} µs"


def main(r="r01"):
    b = load(f"{r}_bench.json")
    pk = b["per_kernel"]
    rows = [
        ("**bitonic 2^24, B=64, 16 keys/thread** (headline)", "bitonic", "melded_frac_hbm", "HBM"),
        ("bitonic 2^24, B=64, one key/thread", "bitonic_1key", "melded_frac_hbm", "HBM"),
        ("bitonic 2^24, B=256 / 1024 / 4096, 16 keys/thread", None, None, None),
        ("sb1 … nested (9 kernels), 2^20 lanes", None, None, None),
        ("NQU N=16, mirror symmetry", "nqueens16", None, None),
        ("PCM 2^24, B=64, 16 keys/thread", "pcm", "melded_frac_hbm", "HBM"),
        ("PCM 2^24, B=64, one key/thread", "pcm_1key", "melded_frac_hbm", "HBM"),
        ("MS 2^20", "ms1m", "melded_frac_hbm", "HBM (L2-resident)"),
        ("LUD 8192²", "lud8192", "melded_frac_fp32", "FP32"),
        ("SRAD 16384² × 100", "srad16384x100", "melded_frac_hbm", "HBM"),
        ("SRAD 16384² × 100, `DARM_FAST_MATH`", "srad16384x100_fast_math", "melded_frac_hbm", "HBM"),
    ]
    print("| kernel | unmelded | melded | speedup | melded vs roof |")
    print("|---|---|---|---|---|")
    for label, key, fk, roof in rows:
        if key is None and label.startswith("bitonic"):
            cells = [pk[f"bitonic_B{B}"] for B in (256, 1024, 4096)]
            unm = " / ".join(t(c["unmelded_us"]) for c in cells)
            mel = " / ".join(t(c["melded_us"]) for c in cells)
            sps = " / ".join(f"{c['speedup']:.2f}×" for c in cells)
            fr = " / ".join(f"{c['roofline']['frac']:.2f}" for c in cells)
            print(f"| {label} | {unm} | {mel} | {sps} | {fr} HBM |")
            continue
        if key is None:
            names = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested"]
            cs = [pk[n] for n in names]
            print(f"| {label} | {min(c['unmelded_us'] for c in cs):.1f}–{max(c['unmelded_us'] for c in cs):.1f} µs | "
                  f"{min(c['melded_us'] for c in cs):.1f}–{max(c['melded_us'] for c in cs):.1f} µs | "
                  f"{min(c['speedup'] for c in cs):.2f}–{max(c['speedup'] for c in cs):.2f}× | "
                  f"{min(c['roofline']['frac'] for c in cs):.2f}–{max(c['roofline']['frac'] for c in cs):.2f} HBM (latency-bound) |")
            continue
        c = pk[key]
        if key == "nqueens16":
            frac = f"{c['roofline']['frac']:.2f} issue"
        else:
            frac = f"{c['roofline']['frac']:.2f} {roof}"
        sp = c["speedup"]
        print(f"| {label} | {t(c['unmelded_us'])} | **{t(c['melded_us'])}** | {sp:.2f}× | {frac} |")
    print()
    le = json.load(open(os.path.join(ROOT, "profiles", f"{r}_lane_efficiency.json")))["kernels"]
    import glob

    sim_path = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9][0-9]_simulator_util.json")))[-1]
    sim = json.load(open(sim_path))["utilization"]
    print("| kernel | reference simulator utilisation (unit latency) unmelded → melded | ncu thread_inst/(32·inst) | "
          "ncu pred_on/(32·inst) | branch uniformity % | warp instructions melded / unmelded | "
          "predicated compile: pred_on/(32·inst), branch uniformity % |")
    print("|---|---|---|---|---|---|---|")
    for k, e in sorted(le.items()):
        u, m = e["unmelded"], e["melded"]
        p = e.get("predicated")
        s = sim.get(k)
        ss = f"{s['unmelded']:.3f} → {s['melded']:.3f}" if s else "—"
        ps = f"{p['lane_efficiency_pred_on']:.3f}, {p['branch_uniform_pct']:.0f}" if p else "—"
        print(f"| {k} | {ss} | {u['lane_efficiency']:.3f} → {m['lane_efficiency']:.3f} | "
              f"{u['lane_efficiency_pred_on']:.3f} → {m['lane_efficiency_pred_on']:.3f} | "
              f"{u['branch_uniform_pct']:.0f} → {m['branch_uniform_pct']:.0f} | {m['warp_inst'] / u['warp_inst']:.2f} | {ps} |")


if __name__ == "__main__":
    main(*sys.argv[1:])
