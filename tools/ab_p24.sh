# A/B of the p24 / c2 bench steps (single filters through the cooperative kernel): in-tree library vs _variants/base.so
mkdir -p gpurun_out/$1
for r in 1 2; do
for w in p24 c2; do
python bench.py --workload $w --steps 10 --warmup 3 --no-extras > gpurun_out/$1/new_${w}_$r.json 2>/dev/null
PF_LIB_OVERRIDE=_variants/base.so python bench.py --workload $w --steps 10 --warmup 3 --no-extras > gpurun_out/$1/base_${w}_$r.json 2>/dev/null
done
done
for f in gpurun_out/$1/*.json; do python -c "
import json
d=json.load(open('$f')); print('$f', d['ms_per_step'], json.dumps({k: round(v['avg_ms'], 4) for k, v in (d.get('kernels') or {}).items()}))"; done
