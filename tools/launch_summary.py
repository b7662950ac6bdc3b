"""Per-kernel totals from an `ncu --metrics ... --csv --log-file` launch list.

    python tools/launch_summary.py gpurun_out/launches.csv
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ni, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    per = defaultdict(lambda: defaultdict(float))
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6,
                 "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(unit, 1.0)
        per[r[ii]][r[ni]] = v * scale
        names[r[ii]] = r[ki][:80]
    agg = defaultdict(lambda: defaultdict(float))
    cnt = defaultdict(int)
    for i, m in per.items():
        cnt[names[i]] += 1
        for k, v in m.items():
            agg[names[i]][k] += v
    print(f"{'launches':>8} {'ms total':>10} {'ms avg':>8} {'GB avg':>8}  kernel")
    for name, m in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
        t = m.get("gpu__time_duration.sum", 0.0)
        gb = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        c = cnt[name]
        print(f"{c:8d} {t:10.3f} {t / c:8.3f} {gb / c:8.3f}  {name}")


if __name__ == "__main__":
    main(sys.argv[1])
