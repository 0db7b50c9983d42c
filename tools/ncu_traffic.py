"""DRAM traffic of one fitness evaluation per workload, from an ncu launch list -> profiles/dram_traffic.json.

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/eval_c4.csv python tools/probe_eval.py c4
    python tools/ncu_traffic.py gpurun_out/eval_c4.csv c4 profiles/r02_eval_c4.csv

Sums dram__bytes_read + dram__bytes_write over every kernel of the ONE evaluation the probe brackets (the clear of the
reached records is a kernel, k_pc_clear, so it is included), copies the launch list under profiles/ and records
{workload: {bytes, kernel_ms, launches, source}} in profiles/dram_traffic.json, which bench.py reads for
roofline.traffic."""
import csv
import json
import os
import shutil
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kernel_base(full):
    """'k<(int)1024>(const int *, ...)' -> 'k<(int)1024>': drop the trailing parameter list only"""
    full = full.strip()
    if not full.endswith(")"):
        return full
    depth = 0
    for i in range(len(full) - 1, -1, -1):
        depth += full[i] == ")"
        depth -= full[i] == "("
        if depth == 0:
            return full[:i].replace("void ", "").replace("gapa_b200::", "")
    return full


def parse(path):
    rows = []
    with open(path, newline="") as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per = defaultdict(lambda: {"ms": 0.0, "bytes": 0.0, "launches": set()})
    for r in rows:
        name = kernel_base(r["Kernel Name"])
        unit, val = r["Metric Unit"], float(r["Metric Value"].replace(",", ""))
        m = r["Metric Name"]
        e = per[name]
        e["launches"].add(r["ID"])
        if m == "gpu__time_duration.sum":
            e["ms"] += val * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}.get(unit, 1e-6)
        elif m.startswith("dram__bytes"):
            e["bytes"] += val * {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1.0)
    return per


def main():
    src, workload = sys.argv[1], sys.argv[2]
    dst = sys.argv[3] if len(sys.argv) > 3 else None
    per = parse(src)
    total_b = sum(e["bytes"] for e in per.values())
    total_ms = sum(e["ms"] for e in per.values())
    for name, e in sorted(per.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"{name:48s} x{len(e['launches']):3d}  {e['ms']:8.4f} ms  {e['bytes'] / 1e9:7.3f} GB  "
              f"{(e['bytes'] / 1e9) / (e['ms'] * 1e-3) if e['ms'] else 0:8.1f} GB/s")
    print(f"{'TOTAL':48s}       {total_ms:8.4f} ms  {total_b / 1e9:7.3f} GB")
    if dst:
        shutil.copyfile(src, os.path.join(ROOT, dst))
        path = os.path.join(ROOT, "profiles", "dram_traffic.json")
        try:
            doc = json.load(open(path))
        except Exception:
            doc = {}
        doc[workload] = {"bytes": total_b, "kernel_ms_under_ncu": total_ms, "launches": sum(len(e["launches"]) for e in per.values()),
                         "source": dst,
                         "kernels": {n: {"ms": round(e["ms"], 5), "gbytes": round(e["bytes"] / 1e9, 4)} for n, e in per.items()}}
        json.dump(doc, open(path, "w"), indent=1, sort_keys=True)
        print("wrote", path)


if __name__ == "__main__":
    main()
