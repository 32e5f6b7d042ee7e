# A/B of the default quick times (C3 steps and single filters of 2^17..2^24): in-tree library vs _variants/base.so
mkdir -p gpurun_out/$1
for r in 1 2; do
python tools/quick_times.py > gpurun_out/$1/dnew_$r.jsonl 2>&1
PF_LIB_OVERRIDE=_variants/base.so python tools/quick_times.py > gpurun_out/$1/dbase_$r.jsonl 2>&1
done
for f in dnew_1 dbase_1 dnew_2 dbase_2; do python -c "
import json
print('$f', ' '.join(str(json.loads(l)['ms']) for l in open('gpurun_out/$1/$f.jsonl')))"; done
