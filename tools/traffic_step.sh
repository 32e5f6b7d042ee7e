# DRAM bytes + duration of the C3 step kernel for each library variant given (ncu metrics only)
for v in "$@"; do
  echo "== $v"
  PF_LIB_OVERRIDE=_variants/$v.so timeout 200 python tools/quick_times.py --c3 | grep systematic | grep step
  PF_LIB_OVERRIDE=_variants/$v.so timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_fused_sorted -s 2 -c 1 --csv python tools/prof_step.py systematic 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
