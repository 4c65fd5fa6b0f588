"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name, count / total / mean.

usage: python tools/launch_list_summary.py launches.csv [first_id [last_id]]
"""
import csv, sys, collections, re


def rows_of(path):
    with open(path, newline="") as f:
        lines = [l for l in f if not l.startswith("==")]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(unit.replace("second", "s").replace("usecond", "us"), 1e-3)
        yield int(r["ID"]), r["Kernel Name"], val * scale


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = re.sub(r"^void ", "", name)
    m = re.match(r"([A-Za-z_0-9:]+)(<[^(]*)?", name)
    base = m.group(1).split("::")[-1] if m else name
    targs = ""
    if m and m.group(2):
        if base.startswith(("ttm_", "gram_")):
            targs = m.group(2)[:24]
        elif base == "Kernel2":
            targs = m.group(2).replace("<cutlass_80_tensorop_", "<")[:40]
    return (base + targs)[:64]


def main():
    path = sys.argv[1]
    lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 60
    agg = collections.OrderedDict()
    total = 0.0
    n = 0
    for i, name, us in rows_of(path):
        if not (lo <= i <= hi):
            continue
        a = agg.setdefault(short(name), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += us
        a[2] = max(a[2], us)
        total += us
        n += 1
    print(f"{n} launches, {total / 1e3:.3f} ms (ids {lo}..{hi if hi < 1 << 60 else 'end'})")
    for name, (cnt, us, mx) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {name:60s} n={cnt:5d} total={us / 1e3:9.3f} ms  mean={us / cnt:9.1f} us  max={mx:9.1f} us  {100 * us / total:5.1f}%")


if __name__ == "__main__":
    main()
