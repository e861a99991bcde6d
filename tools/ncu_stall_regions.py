"""Warp-stall samples of one kernel in an ncu report, bucketed: the DMMA k-loop clusters vs the
rest, and by opcode / stall reason (SASS source page). Usage:
    python tools/ncu_stall_regions.py report.ncu-rep <kernel regex> [launch index]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, kre, idx="0"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kre}", "--launch-skip", idx, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    body = [r for r in rows[2:] if len(r) > 10]
    si = h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]

    def I(x):
        try:
            return int(x)
        except ValueError:
            return 0
    tot = sum(I(r[si]) for r in body)
    dm = [i for i, r in enumerate(body) if "DMMA" in r[1]]
    inside = set()
    if dm:
        s = p = dm[0]
        for i in dm[1:] + [10 ** 9]:
            if i - p > 60:
                inside.update(range(s, p + 1))
                s = i
            p = i
    ins = sum(I(body[i][si]) for i in inside)
    print(f"samples {tot}; in DMMA k-loop clusters {100 * ins / tot:.1f} %, elsewhere {100 * (tot - ins) / tot:.1f} %")
    op = collections.Counter()
    rs = collections.Counter()
    for r in body:
        t = r[1].split()
        if t:
            op[t[1] if t[0].startswith("@") else t[0]] += I(r[si])
        for c in reasons:
            rs[c[6:]] += I(r[h.index(c)])
    print("by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}" for k, v in op.most_common(8)))
    print("by reason:", ", ".join(f"{k} {100 * v / tot:.1f}" for k, v in rs.most_common(8)))


if __name__ == "__main__":
    main(*sys.argv[1:])
