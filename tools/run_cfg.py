"""Run fpe_evaluate on one BASELINE config a few times (a target for ncu and quick timing):

    python tools/run_cfg.py --config 5 --fp32 --steps 3 [--points N]

Prints per-stage CUDA-event times of the last step (library profiling events).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--fp32", action="store_true")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--points", type=int, default=0)
    args = ap.parse_args()
    import torch

    import paper_2211_06320_b200 as fpe
    import workloads
    a = workloads.coefficients(args.config)
    p = workloads.points(args.config, args.points or None)
    if args.fp32:
        a, p = workloads.to_fp32(a), workloads.to_fp32(p)
    poly = fpe.precondition(a)
    pts = torch.from_numpy(p).cuda()
    del p
    for _ in range(args.steps):
        poly.evaluate(pts, exps=True)
    poly.set_profiling(True)
    poly.evaluate(pts, exps=True)
    st = poly.last_stage_ms()
    poly.set_profiling(False)
    poly.evaluate(pts, exps=True)
    print(json.dumps({"config": args.config, "fp32": args.fp32, "points": pts.numel(), "stages_ms": st,
                      "total_ms": sum(t for _, t in st), "counters": poly.workspace_stats()}))


if __name__ == "__main__":
    main()
