"""Device time of one fpe_evaluate over 2^26 cfg3 points vs the same points as sub-batches (slices) on one
stream or round-robin over several streams (each with its own workspace) -- does keeping a sub-batch's
records L2-resident pay for the per-batch fixed costs?"""
import sys
import torch

sys.path[:0] = ['.']
import paper_2211_06320_b200 as fpe  # noqa: E402
import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
poly = fpe.precondition(workloads.coefficients(cfg))
n = workloads.CONFIGS[cfg]["n_points"] if cfg != 5 else 1 << 26
pts = torch.from_numpy(workloads.points(cfg, n)).cuda()
vals = torch.empty(n, dtype=torch.complex128, device="cuda")
exps = torch.empty(n, dtype=torch.int64, device="cuda")


def timed(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ws_full = poly.workspace(n)
print("whole batch", round(timed(lambda: poly.evaluate(pts, out=vals, workspace=ws_full)), 3), flush=True)
del ws_full
torch.cuda.empty_cache()
for lg in (21, 22, 23, 24):
    m = 1 << lg
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        wss = [poly.workspace(m, streams[i]) for i in range(ns)]
        cur = torch.cuda.current_stream()

        def run():
            ev = torch.cuda.Event()
            ev.record(cur)
            for s in streams:
                s.wait_event(ev)
            for i, lo in enumerate(range(0, n, m)):
                s = streams[i % ns]
                with torch.cuda.stream(s):
                    poly.evaluate(pts[lo:lo + m], out=vals[lo:lo + m], workspace=wss[i % ns])
            for s in streams:
                e2 = torch.cuda.Event(); e2.record(s); cur.wait_event(e2)
        print(f"slices 2^{lg} on {ns} stream(s)", round(timed(run), 3), flush=True)
        del wss
        torch.cuda.empty_cache()
