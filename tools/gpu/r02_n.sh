#!/bin/bash
# round 2, call n (1 GPU): real-split CTA raster (group rows) timings + DRAM bytes per launch
mkdir -p gpurun_out/r02n
for G in 0 2 4 8 16; do
  BSE200_RS_GROUP_ROWS=$G timeout 600 python tools/rs_bench.py 20000 1200,300 90 2>&1 | sed "s/^/G=$G /"
done | tee gpurun_out/r02n/rs_raster.txt
for G in 0 8; do
  BSE200_RS_GROUP_ROWS=$G timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:hop_rs_tma_kernel -c 2 python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02n/ncu_raster_G$G.txt 2>&1
  grep -E "dram__bytes|gpu__time|lts__t_sector_hit|dmma_cycles" gpurun_out/r02n/ncu_raster_G$G.txt | head -10
done
