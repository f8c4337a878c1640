"""Warp-stall breakdown of one kernel in an ncu report (source page, SASS level):
overall stall reasons and the hottest instructions with their top reasons."""
import collections
import csv
import io
import subprocess
import sys


def main(path, ntop=20):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, rows = r[1], r[2:]
    I, S, E, A = (h.index(k) for k in ("Source", "Warp Stall Sampling (All Samples)", "Instructions Executed", "Address"))
    st = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    rows = [x for x in rows if x[S].isdigit()]
    tot = collections.Counter()
    ops = collections.Counter()
    n_exec = 0
    for x in rows:
        n_exec += int(x[E] or 0)
        for i in st:
            if x[i].isdigit():
                tot[h[i]] += int(x[i])
        f = x[I].split()
        if f:
            op = f[1] if f[0].startswith("@") and len(f) > 1 else f[0]
            ops[op.split(".")[0]] += int(x[E] or 0)
    T = sum(tot.values())
    print(f"warp instructions executed {n_exec}, stall samples {T}")
    print("stall reasons:", ", ".join(f"{k[6:]} {v / T * 100:.1f}%" for k, v in tot.most_common(10)))
    print("instruction mix:", ", ".join(f"{k} {v / n_exec * 100:.1f}%" for k, v in ops.most_common(14)))
    for x in sorted(rows, key=lambda x: -int(x[S]))[:ntop]:
        rs = sorted([(int(x[i]), h[i][6:]) for i in st if x[i].isdigit() and int(x[i]) > 0], reverse=True)[:3]
        print(f"  {x[A][-5:]} {int(x[S]) / T * 100:5.1f}% exec={x[E]:>8} {x[I].strip()[:48]:48s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
