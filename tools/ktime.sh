#!/bin/bash
# per-kernel launch list of one bench frame: tools/ktime.sh TAG  (run on the GPU box)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-comparator > gpurun_out/ncu_$1.log 2>&1
