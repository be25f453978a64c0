"""Summarise an ncu --csv launch list (gpu__time_duration.sum, optionally dram bytes) per kernel family.
Usage: python scripts/summarize_ncu_csv.py launches.csv [--per-launch]"""
import collections
import csv
import sys


def rows(path):
    data = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(data) if r and r[0] == "ID"][0]
    hdr = data[hi]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = collections.OrderedDict()
    for r in data[hi + 1:]:
        if len(r) > vi:
            launches.setdefault(r[0], {"kernel": r[ki]})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    return list(launches.values())


def family(name):
    n = name.split("(")[0].replace("void ", "")
    return n if "<" not in n else n.split("<")[0] + "<" + n.split("<")[1].split(">")[0] + ">"


def main(path, per_launch=False):
    ls = rows(path)
    tot = sum(l["gpu__time_duration.sum"][0] for l in ls)
    print(f"{len(ls)} launches, sum of kernel durations {tot / 1e3:.1f} us ({path})")
    agg = collections.OrderedDict()
    for l in ls:
        a = agg.setdefault(family(l["kernel"]), [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += l["gpu__time_duration.sum"][0]
        a[2] += l.get("dram__bytes_read.sum", (0, ""))[0]
        a[3] += l.get("dram__bytes_write.sum", (0, ""))[0]
    print(f"{'kernel':60s} {'n':>4s} {'us':>9s} {'share':>6s} {'us/launch':>9s} {'DRAM GB/s':>9s}")
    for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = (rd + wr) / t if t else 0.0        # bytes / ns = GB/s
        print(f"{k[:60]:60s} {n:4d} {t / 1e3:9.1f} {100 * t / tot:5.1f}% {t / n / 1e3:9.2f} {gbs:9.1f}")
    if per_launch:
        for l in ls:
            print(family(l["kernel"])[:60], l["gpu__time_duration.sum"][0] / 1e3)


if __name__ == "__main__":
    main(sys.argv[1], "--per-launch" in sys.argv)
