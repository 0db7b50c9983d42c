for cfg in "GAPA_PC_SPEC_ROUNDS=0" "GAPA_PC_SPEC_ROUNDS=1"; do
for wp in "n1e4 256" "n1e4 4096" "n1e5 4096" "n1e5 16384" "c1 0"; do set -- $wp
  echo "== $cfg $1 pop $2"
  env $cfg python bench.py --workload $1 --pop $2 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.4f ms  eval %.4f ms  vary+eval %.4f ms  launches %d  loop %.1f gen/s' % (d['ms_per_step'], d['fitness_eval_ms_per_step'], d['variation_plus_eval_ms_per_step'], d['gpu_launches'], d.get('library_loop',{}).get('generations_per_sec',0)))
    elif l: print(l[:300])
"
done; done
