"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: launches,
total device time, share. Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        except ValueError:
            continue
        name = r[ik].split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot:.1f} ms over {sum(v[0] for v in agg.values())} launches (cold-cache, serialised by ncu)")
    for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:6d} {ms:12.3f} ms {100 * ms / tot:6.2f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
