set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-comparator --no-configs --no-ncu > gpurun_out/b_pre.json 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "riann_bench_frame/" -k regex:"bulk_p0_kernel|bulk_final|bulk_filter" -c 3 -o gpurun_out/r2_full python bench.py --ncu-child --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
