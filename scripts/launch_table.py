"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) for
one step: the launches between the last two gather kernels, grouped by
kernel.  Usage: python scripts/launch_table.py launches.csv [--per-launch]"""
import collections
import csv
import sys


def load(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def short(n):
    n = n.split("(")[0].replace("void ", "")
    for p in ("attn::<unnamed>::", "kern::<unnamed>::", "gemm::"):
        n = n.replace(p, "")
    return n


def main():
    data = load(sys.argv[1])
    idx = [i for i, d in enumerate(data)
           if "gather_batch" in d["Kernel Name"] or "gather_tokens" in d["Kernel Name"]]
    st, en = (idx[-2], idx[-1]) if len(idx) >= 2 else (idx[-1], len(data))
    step = data[st:en]
    agg = collections.OrderedDict()
    for d in step:
        a = agg.setdefault(short(d["Kernel Name"]), [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"{'us':>10} {'share':>6} {'n':>4}  kernel")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v:10.1f} {100 * v / tot:5.1f}% {c:4d}  {n}")
    print(f"{tot:10.1f}  total (one step, {len(step)} launches; ncu-serialised, cold-cache)")
    if "--per-launch" in sys.argv:
        for d in step:
            print(f"{float(d['Metric Value']) / 1e3:9.1f} us  {short(d['Kernel Name'])}")


if __name__ == "__main__":
    main()
