"""Summarise an `ncu --page source --csv --print-source=sass` dump: instruction share, average active
threads and top opcodes per region of N SASS lines (profiling helper)."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        try:
            float(r[h.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        data.append(r)
    return h, data


def main(path, width=64, thresh=0.015):
    h, data = load(path)
    iS, iE, iT = h.index("Source"), h.index("Instructions Executed"), h.index("Avg. Threads Executed")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    idx = [h.index(c) for c in cols]
    ws = [sum(float(r[j] or 0) for j in idx) for r in data]
    tot = sum(float(r[iE] or 0) for r in data)
    TW = sum(ws) or 1
    print("rows", len(data), "instructions", tot)
    for s in range(0, len(data), width):
        blk = data[s:s + width]
        e = sum(float(r[iE] or 0) for r in blk)
        w = sum(ws[s:s + width])
        if e / tot < thresh and w / TW < thresh:
            continue
        ops = {}
        for r in blk:
            t = r[iS].split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[op] = ops.get(op, 0) + float(r[iE] or 0)
        top = sorted(ops.items(), key=lambda x: -x[1])[:6]
        thr = sum(float(r[iE] or 0) * float(r[iT] or 0) for r in blk) / max(e, 1)
        print(f"{s:6d} exec {e / tot * 100:5.1f}% stall {w / TW * 100:5.1f}% thr={thr:4.1f}",
              [(k, round(v / max(e, 1) * 100)) for k, v in top])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 64)
