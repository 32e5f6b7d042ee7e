# A/B of the C3 quick times: the in-tree library against _variants/base.so, alternated twice
mkdir -p gpurun_out/$1
for r in 1 2; do
python tools/quick_times.py --c3 > gpurun_out/$1/new_$r.jsonl 2>&1
PF_LIB_OVERRIDE=_variants/base.so python tools/quick_times.py --c3 > gpurun_out/$1/base_$r.jsonl 2>&1
done
for f in new_1 base_1 new_2 base_2; do python -c "
import json
print('$f', ' '.join(str(json.loads(l)['ms']) for l in open('gpurun_out/$1/$f.jsonl')))"; done
