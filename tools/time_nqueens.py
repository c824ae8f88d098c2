"""Time N-Queens (both forms) on cuda:0 for a few prefix depths (run under gpurun)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402


def main(n=16, mirror=1):
    darm.init()
    for base in (5, 6, 7, 8, 9):
        row = {}
        for v in (darm.UNMELDED, darm.MELDED):
            ts = []
            for i in range(6):
                sols, _, st = darm.nqueens(n, base, v, mirror=bool(mirror))
                assert sols == {15: 2279184, 16: 14772512, 17: 95815104}[n], sols
                if i >= 2:
                    ts.append(st["kernel_ms"])
            row[v] = min(ts)
        print(f"n={n} mirror={mirror} base={base} unmelded {row[0]:.3f} ms melded {row[1]:.3f} ms speedup {row[0] / row[1]:.3f}",
              flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
