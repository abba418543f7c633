# K4 timing probes: kernel-only duration (ncu, gpu__time_duration) of exact_tc_kernel for the full kernel,
# the epilogue alone (no MMA issued) and the MMA pipeline alone (no TMEM reads), 2 waves of CTAs
for cfg in 3 4; do for v in k4pipe k4nomma k4noepi; do
  echo "== cfg$cfg $v"
  RIANN_LIB=$PWD/_ab/lib_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:exact_tc_kernel --csv \
    python tools/bench_exact.py --cfg $cfg --m 37888 --simt-m 64 --reps 1 2>/dev/null | grep exact_tc_kernel | awk -F'","' '{print $NF}'
done; done
