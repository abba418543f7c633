# ncu --set full of the final-scan kernel (and P0a/draw/window) of the last frame of a short bench run
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "riann_bench_frame/" -k regex:"bulk_final" -c 1 -o gpurun_out/r2_final python bench.py --ncu-child --steps 2 --warmup 3 > gpurun_out/ncu_final.log 2>&1
echo ncu_rc=$?
