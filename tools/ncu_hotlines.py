"""Top source lines (instructions executed, warp-stall samples) of one kernel in an ncu report:
    python tools/ncu_hotlines.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(path, kregex, top=30):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=cuda,sass", "-k",
                          f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    cur, out, h = None, [], None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if h is None or len(r) < 8 or r[2] != "-":
            continue
        try:
            e, w = float(r[7] or 0), float(r[4] or 0)
        except ValueError:
            continue
        out.append((e, w, cur, r[0], r[1][:110]))
    tot = sum(o[0] for o in out) or 1
    totw = sum(o[1] for o in out) or 1
    byf = collections.Counter()
    for o in out:
        byf[o[2]] += o[0]
    print(f"{kregex}: {tot:.4g} warp instructions; by file: " +
          ", ".join(f"{f} {100 * v / tot:.1f}%" for f, v in byf.most_common()))
    for e, w, f, ln, s in sorted(out, key=lambda x: -x[1])[:top]:
        print(f"{100 * e / tot:5.1f}% instr {100 * w / totw:5.1f}% stalls  {f}:{ln}: {s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
