"""Summarise an ncu launch-list CSV (gpu__time_duration.sum, dram__bytes_read/write.sum per launch) of one train
step: per kernel family -> launches, time, share, DRAM bytes and achieved GB/s (vs the measured HBM peak).

    python scripts/ncu_summary.py gpurun_out/r2i_launches_650m.csv [--hbm 6529.4] > profiles/....txt
"""
import argparse
import collections
import csv
import re


def family(name: str) -> str:
    n = re.sub(r"\(.*", "", name.replace("void ", ""))
    n = re.sub(r"<.*", "", n)
    return n.strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--hbm", type=float, default=6529.4)
    ap.add_argument("--step-marker", default="mlm_mask_kernel")
    a = ap.parse_args()
    rows = collections.OrderedDict()
    with open(a.csv) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        k = int(r["ID"])
        d = rows.setdefault(k, {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ns"] = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        else:
            d[r["Metric Name"]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    ids = list(rows)
    starts = [i for i in ids if a.step_marker in rows[i]["name"]]
    if starts:  # the last complete step: from the last-but-one marker (or first) to the next marker / end
        s0 = starts[0]
        s1 = starts[1] if len(starts) > 1 else ids[-1] + 1
        ids = [i for i in ids if s0 <= i < s1]
    fam = collections.OrderedDict()
    for i in ids:
        d = rows[i]
        f = fam.setdefault(family(d["name"]), {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
        f["n"] += 1
        f["ns"] += d.get("ns", 0.0)
        f["rd"] += d.get("dram__bytes_read.sum", 0.0)
        f["wr"] += d.get("dram__bytes_write.sum", 0.0)
    tot = sum(f["ns"] for f in fam.values())
    print(f"# {a.csv}: launches {ids[0]}..{ids[-1]} ({len(ids)} kernels, one step), total {tot / 1e6:.3f} ms "
          f"(serialised, cold-cache ncu replay timing)")
    print(f"{'kernel':58s} {'n':>4s} {'ms':>8s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>7s} {'frac_HBM':>8s}")
    for k, f in sorted(fam.items(), key=lambda kv: -kv[1]["ns"]):
        mb = (f["rd"] + f["wr"]) / f["n"] / 1e6
        gbs = (f["rd"] + f["wr"]) / f["ns"] if f["ns"] else 0.0
        print(f"{k[:58]:58s} {f['n']:4d} {f['ns'] / 1e6:8.3f} {f['ns'] / tot:6.3f} {mb:10.1f} {gbs:7.0f} "
              f"{gbs / a.hbm:8.3f}")


if __name__ == "__main__":
    main()
