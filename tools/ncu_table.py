"""Summarise an `ncu --csv --metrics ...` launch log: one row per kernel
launch (or the median per kernel name with --median)."""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    launches = collections.OrderedDict()
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        d = launches.setdefault(r[ii], {"kernel": r[ki]})
        d[r[mi]] = v
    return list(launches.values())


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("emoe::", "")
    return name.split("(")[0][:48]


if __name__ == "__main__":
    ls = load(sys.argv[1])
    keys = [k for k in ls[0] if k != "kernel"]
    print(f"{'kernel':48s} " + " ".join(f"{k.split('.')[0].split('__')[-1][:14]:>14s}" for k in keys))
    for d in ls:
        print(f"{short(d['kernel']):48s} " + " ".join(f"{d.get(k, 0):14.1f}" for k in keys))
