#!/bin/bash
# per-kernel device time of the c4 fused step (ncu launch list, warm caches)
python tools/c4_step.py > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -s 60 -c 120 --csv --log-file gpurun_out/c4launch.csv python tools/c4_step.py > /dev/null 2>&1
cat gpurun_out/plain.log
