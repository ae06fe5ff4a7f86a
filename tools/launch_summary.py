"""Summarize an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel
count / total / mean for the last `--steps` profiled steps (the script runs
warm-up steps first, so the tail fraction is the measured step)."""
import collections
import csv
import sys


def main(path, frac=0.5):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tail = data[int(len(data) * (1 - frac)):]
    agg = collections.OrderedDict()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for d in tail:
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        v = float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'total us':>10} {'count':>5} {'mean us':>10} {'share':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {c:5d} {t / c:10.1f} {100 * t / tot:5.1f}%  {k}")
    print(f"{tot:10.1f} us total over {len(tail)} launches")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.5)
