#!/bin/bash
# round 2: DRAM bytes per launch of the default real-split tile vs the CTA raster's row-tile group
# (BSE200_RS_GROUP_ROWS) at C3, k = 1200 -- time from rs_bench (no profiler), bytes from ncu
mkdir -p gpurun_out/r02r
for G in 8 16 32 64; do
  BSE200_RS_GROUP_ROWS=$G timeout 300 python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02r/rs_G$G.jsonl 2>&1
  BSE200_RS_GROUP_ROWS=$G timeout 600 ncu --clock-control none -k regex:hop_rs_tma_kernel -c 1 --csv \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,launch__grid_size \
    python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02r/ncu_G$G.csv 2>&1
  echo "G=$G $(tail -1 gpurun_out/r02r/rs_G$G.jsonl | cut -c1-200)"; grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/r02r/ncu_G$G.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
