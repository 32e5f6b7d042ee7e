set -x
mkdir -p gpurun_out/m
python bench.py --steps 20 --warmup 5 > gpurun_out/m/bench_c3.json 2> gpurun_out/m/bench_c3.err
for sc in stratified multinomial metropolis; do python bench.py --scheme $sc --steps 10 --warmup 3 --no-extras > gpurun_out/m/bench_$sc.json 2>/dev/null; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_sorted -s 2 -c 1 -o /tmp/step_sys python tools/prof_step.py systematic > gpurun_out/m/ncu_step.log 2>&1
python tools/evidence.py /tmp/step_sys.ncu-rep c3/systematic --source "ncu --set full --clock-control none -k regex:k_fused_sorted -s 2 -c 1 python tools/prof_step.py (round 2 final)" > gpurun_out/m/evidence.log 2>&1
cp profiles/kernel_evidence.json gpurun_out/m/kernel_evidence.json
python tools/ncu_summary.py /tmp/step_sys.ncu-rep > gpurun_out/m/step_summary.md 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_sorted -s 2 -c 1 -o /tmp/ro_sys python tools/prof_resample_only.py systematic > gpurun_out/m/ncu_ro.log 2>&1
python tools/ncu_summary.py /tmp/ro_sys.ncu-rep > gpurun_out/m/ro_summary.md 2>&1
ncu -i /tmp/ro_sys.ncu-rep --page raw --csv > gpurun_out/m/ro_raw.csv 2>/dev/null
ncu -i /tmp/step_sys.ncu-rep --page raw --csv > gpurun_out/m/step_raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m/launches.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/m/ncu_launch.log 2>&1
ls -la gpurun_out/m
python tools/sass_lines.py /tmp/ro_sys.ncu-rep k_fused_sorted k_fused_sortedILi3ELb0ELi0ELi256 --outer --top 60 > gpurun_out/m/ro_sys_outer.txt 2>&1
python tools/sass_lines.py /tmp/ro_sys.ncu-rep k_fused_sorted k_fused_sortedILi3ELb0ELi0ELi256 --top 60 > gpurun_out/m/ro_sys_lines.txt 2>&1
python tools/sass_lines.py /tmp/step_sys.ncu-rep k_fused_sorted k_fused_sortedILi3ELb0ELi2ELi512ELi16ELb0 --outer --top 60 > gpurun_out/m/step_outer.txt 2>&1
