"""SRAD 16384^2 x 100 kernel time, both forms, IEEE and DARM_FAST_MATH."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2107_05681_b200 as d  # noqa: E402

d.init()
n = 16384
g = torch.Generator(device="cuda").manual_seed(5)
j0 = torch.exp(torch.rand((n, n), generator=g, device="cuda"))
j = torch.empty_like(j0)
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for fast in (False, True):
    r = {}
    for v in (0, 1):
        ts = []
        for i in range(3):
            j.copy_(j0)
            st = d.srad(j, 100, 0.5, d.RODINIA_ROI, v, fast=fast)
            if i:
                ts.append(st["kernel_ms"])
        r[v] = min(ts)
    print(tag, "fast", fast, "unmelded %.1f ms melded %.1f ms speedup %.3f" % (r[0], r[1], r[0] / r[1]), flush=True)
