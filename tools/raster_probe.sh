#!/bin/bash
# DRAM bytes and time of the fused kernel against the rasterisation group (STC_GROUP_M): tools/raster_probe.sh bar 2 abc
cfg=${1:-bar}; lvl=${2:-2}; var=${3:-abc}
mkdir -p gpurun_out
for g in ${GROUPS_M:-4 8 12 16 32}; do
  echo "== STC_GROUP_M=$g"
  STC_GROUP_M=$g python tools/one_call.py $cfg $lvl $var 3
  STC_GROUP_M=$g ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_strassen_fused -c 1 --csv python tools/one_call.py $cfg $lvl $var 1 2>/dev/null | grep -E "dram__|gpu__time|hit_rate" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
