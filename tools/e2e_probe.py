"""e2e of the HOST-mode bitonic sort (2^24 keys, B=64) through the C-ABI (run under gpurun)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402

darm.init()
n = 1 << 24
rng = np.random.default_rng(1)
pristine = rng.integers(-(2 ** 31), 2 ** 31, size=n, dtype=np.int64).astype(np.int32)
host = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
ts = []
for i in range(13):
    host[:] = pristine
    st = darm.bitonic_sort(host, 64, darm.MELDED)
    if i >= 3:
        ts.append(st["total_ms"])
print(os.environ.get("DARM_CHUNK_LOG", "21"), "e2e ms min %.3f mean %.3f  keys/s %.3e" % (min(ts), sum(ts) / len(ts), n / (sum(ts) / len(ts) / 1e3)))
