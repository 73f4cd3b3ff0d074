#!/bin/bash
# DRAM traffic of the large-n FWHT kernel vs chunk size (ncu, cache-control none)
python tools/prof_ff.py fwht 65536 > gpurun_out/plain.log 2>&1 || exit 1
for mb in 2 4 8 16 32; do
  MCK_FWHT_CHUNK_MB=$mb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:fwht_large -s 1 -c 1 --csv python tools/prof_ff.py fwht 65536 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v mb=$mb '{print mb" MB: "$(NF-2)" "$NF}'
done
