#!/bin/bash
# c4 fused-step launch tables for several library builds
for lib in "$@"; do
  echo "== $lib"
  MCK_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -s 60 -c 120 --csv --log-file gpurun_out/ab_launch.csv python tools/c4_step.py > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/ab_launch.csv | head -4
done
