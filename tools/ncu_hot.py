"""Hot instructions of an ncu report's source page (SASS): stall samples and executed counts.

    python tools/ncu_hot.py report.ncu-rep [top]
Prints the top instructions by warp-stall samples with their dominant stall reasons, and the
executed-instruction total per opcode class.
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ix = {n: i for i, n in enumerate(hdr)}
    stall_cols = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
    recs = []
    ops = Counter()
    total_exec = 0
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        try:
            samples = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            ex = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        src = r[ix["Source"]]
        toks = src.split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        ops[op.split(".")[0]] += ex
        total_exec += ex
        st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        recs.append((samples, ex, r[ix["Address"]], src, st))
    tot = sum(x[0] for x in recs) or 1
    recs.sort(key=lambda x: -x[0])
    print(f"total stall samples {tot}, executed warp instructions {total_exec}")
    for s, ex, a, src, st in recs[:top]:
        print(f"{100 * s / tot:5.1f}% {ex:9d} {a:>6} {src[:60]:60s} " + " ".join(f"{n}={v}" for v, n in st if v))
    print("executed by opcode:", ", ".join(f"{k}={v}" for k, v in ops.most_common(25)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
