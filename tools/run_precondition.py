"""Wall time of the host and the device preconditioner (the call only, median of 5) on cfg3 / cfg5 / cfg4."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2211_06320_b200 as fpe
    import workloads
    for cfg in (3, 5, 4):
        a = torch.from_numpy(workloads.coefficients(cfg)).cuda()

        def wall(f, reps=5):
            ts = []
            for _ in range(reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                h = f()
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
                h.close()
            return 1e3 * sorted(ts)[len(ts) // 2], [round(1e3 * t, 2) for t in ts]
        fpe.precondition_gpu(a).close()
        mh, th = wall(lambda: fpe.precondition(a))
        mg, tg = wall(lambda: fpe.precondition_gpu(a))
        print(json.dumps({"cfg": cfg, "host_ms": mh, "gpu_ms": mg, "host_all": th, "gpu_all": tg}))


if __name__ == "__main__":
    main()
