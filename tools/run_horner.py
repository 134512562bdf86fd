"""fpe_horner (full Horner, the context baseline) on cfg3's polynomial: a target for ncu / timing."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2211_06320_b200 as fpe
    import workloads
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
    poly = fpe.precondition(workloads.coefficients(3))
    pts = torch.from_numpy(workloads.points(3, n, shard=5)).cuda()
    for _ in range(2):
        poly.horner(pts)
    poly.set_profiling(True)
    poly.horner(pts)
    st = poly.last_stage_ms()
    ms = sum(t for _, t in st)
    fma = 4.0 * (poly.info["k_max"] - poly.info["k_min"] + 1) * n
    print(json.dumps({"points": n, "ms": ms, "fma_per_s": fma / (ms * 1e-3), "frac": fma / (ms * 1e-3) / (148 * 64 * 1.965e9)}))


if __name__ == "__main__":
    main()
