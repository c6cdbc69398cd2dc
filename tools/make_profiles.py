"""Condense gpurun_out/ ncu artefacts into tracked summaries under profiles/.

python tools/make_profiles.py <round_tag> launches.csv [name=report.ncu-rep ...]
Writes profiles/<tag>_launches.csv (kernel, grid, launches, mean/min us, share of
the run's kernel time), profiles/<tag>_<name>_ncu.json (tools/ncu_summary.py)
and updates profiles/ncu_summary.json {name: {dram_bytes_per_launch, ...}}
(read by bench.py for roofline.traffic)."""
import collections
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.environ.get("TRI_PROF_DIR", os.path.join(ROOT, "profiles"))


def to_bytes(s):
    v, u = s.split()
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        k = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", d["Kernel Name"])
        agg.setdefault((k, d["Grid Size"], d["Block Size"]), []).append(float(d["Metric Value"]) / 1e3)
    total = sum(sum(v) for v in agg.values())
    out = os.path.join(PROF, f"{tag}_launches.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "grid", "block", "launches", "mean_us", "min_us", "share_of_kernel_time"])
        for (k, g, b), v in agg.items():
            w.writerow([k, g, b, len(v), round(sum(v) / len(v), 2), round(min(v), 2), round(sum(v) / total, 4)])
    return out


def main():
    tag, lcsv = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    print(launches(tag, lcsv))
    sp = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(sp)) if os.path.exists(sp) else {}
    for arg in sys.argv[3:]:
        name, rep = arg.split("=", 1)
        s = summarise(rep)
        out = os.path.join(PROF, f"{tag}_{name}_ncu.json")
        json.dump(s, open(out, "w"), indent=1)
        d = s[0]
        summ[name] = {"kernel": d["kernel"], "round": tag,
                      "dram_bytes_per_launch": to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"]),
                      "duration": d["gpu__time_duration.sum"], "source": os.path.basename(out),
                      "inst_per_launch": float(d.get("smsp__inst_executed.sum", "0 inst").split()[0])}
        print(out)
    json.dump(summ, open(sp, "w"), indent=1)


if __name__ == "__main__":
    main()
