"""Condense tools/lambda_vs_bb_ncu.sh output into profiles/<tag>_lambda_vs_bb_ncu.json:
per kernel, the lambda and BB launch counters side by side and the derived waste
(threads launched minus useful predicated-on work is not separable by ncu; we report
threads / warps / CTAs launched, instructions, divergent branch targets)."""
import csv
import glob
import json
import os
import sys


def read(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = None
    out = {}
    for r in rows:
        if r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out["kernel"] = d["Kernel Name"]
            out[d["Metric Name"]] = d["Metric Value"].replace(",", "")
    return out


def main():
    tag, src = sys.argv[1], sys.argv[2]
    res = {}
    for p in sorted(glob.glob(os.path.join(src, "*.csv"))):
        name = os.path.basename(p)[:-4]
        res[name] = read(p)
    pairs = {}
    for name in res:
        if name.endswith("_lambda"):
            base = name[:-7]
            lam, bb = res[name], res.get(base + "_bb", {})
            def f(d, k):
                try:
                    return float(d.get(k, "nan"))
                except ValueError:
                    return float("nan")
            pairs[base] = {"lambda": lam, "bb": bb,
                           "ratio_bb_over_lambda": {k: round(f(bb, k) / f(lam, k), 4) for k in (
                               "gpu__time_duration.sum", "sm__ctas_launched.sum", "smsp__warps_launched.sum",
                               "smsp__threads_launched.sum", "smsp__inst_executed.sum",
                               "smsp__sass_branch_targets_threads_divergent.sum") if f(lam, k) > 0}}
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       f"{tag}_lambda_vs_bb_ncu.json")
    json.dump(pairs, open(out, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
