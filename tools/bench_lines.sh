#!/bin/bash
# Driver-comparable bench lines (both arms) for every workload bench.py knows -> gpurun_out/<tag>_bench_lines.jsonl
TAG=${1:-r02}
OUT=gpurun_out/${TAG}_bench_lines.jsonl
: > $OUT
for w in c4 c1 c2 c3 n1e5 n1e4; do
  python bench.py --workload $w --steps 10 --warmup 3 2>/dev/null | tail -1 >> $OUT
  python bench.py --workload $w --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 >> $OUT
done
python - <<PY
import json
for l in open("$OUT"):
    d = json.loads(l)
    print(d.get("impl", "ours"), d["config"]["workload"][:40], "value %.4g" % d["value"], "ms/step %.4g" % d["ms_per_step"],
          "e2e %.4g" % d["e2e"]["value"], "cpu", d.get("cpu_baseline", {}).get("value"))
PY
