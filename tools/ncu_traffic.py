"""Summarise an ncu CSV launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum, lts__t_bytes.sum) of ONE
reduction: per kernel time/DRAM/L2 bytes, and record the pass kernels' DRAM
bytes per step into profiles/ncu_traffic.json under KEY (bench.py's
roofline.traffic).  usage: python tools/ncu_traffic.py CSV KEY [--write]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    launches = {}
    for r in rows:
        k = (r["ID"], r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                 "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1}.get(unit, 1)
        launches.setdefault(k, {})[r["Metric Name"]] = v * scale
    return launches


def main():
    path, key = sys.argv[1], sys.argv[2]
    L = load(path)
    tot = {"time": 0.0, "dram": 0.0, "l2": 0.0}
    passes = []
    for (i, name), m in sorted(L.items(), key=lambda kv: int(kv[0][0])):
        t = m.get("gpu__time_duration.sum", 0)
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        l2 = m.get("lts__t_bytes.sum", 0)
        short = name.split("(")[0][:60]
        print(f"{i:>4} {short:60s} {t*1e3:10.3f} ms  DRAM {dram/1e9:9.3f} GB  L2 {l2/1e9:9.2f} GB")
        if "pass_v" in name or "pass_flags" in name:
            passes.append({"kernel": short, "ms": t * 1e3, "dram_bytes": dram, "l2_bytes": l2})
            tot["time"] += t
            tot["dram"] += dram
            tot["l2"] += l2
    print(f"pass kernels: {tot['time']*1e3:.1f} ms, DRAM {tot['dram']/1e9:.3f} GB, L2 {tot['l2']/1e9:.1f} GB")
    if "--write" in sys.argv:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = {}
        if os.path.exists(p):
            d = json.load(open(p))
        d = {k: v for k, v in d.items() if k.count(":") == 4}  # current key format only
        d[key] = tot["dram"]
        d.setdefault("_per_pass", {})[key] = passes
        json.dump(d, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
