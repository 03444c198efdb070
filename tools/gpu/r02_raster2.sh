#!/bin/bash
# round 2: DRAM bytes vs raster group at G = 2 / 4 (split-K plan at C3, k = 1200), unsplit G = 8 for
# reference, and one ncu --set full capture of the default plan's product
mkdir -p gpurun_out/r02r
for G in 2 4; do
  BSE200_RS_GROUP_ROWS=$G timeout 300 python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02r/rs_G$G.jsonl 2>&1
  BSE200_RS_GROUP_ROWS=$G timeout 600 ncu --clock-control none -k regex:hop_rs_tma_kernel -c 1 --csv \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,launch__grid_size \
    python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02r/ncu_G$G.csv 2>&1
  echo "G=$G $(tail -1 gpurun_out/r02r/rs_G$G.jsonl | cut -c1-200)"; grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/r02r/ncu_G$G.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
BSE200_RS_KSPLIT=1 timeout 600 ncu --clock-control none -k regex:hop_rs_tma_kernel -c 1 --csv \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,launch__grid_size \
    python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02r/ncu_G8_nosplit.csv 2>&1
echo "G=8 unsplit"; grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/r02r/ncu_G8_nosplit.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hop_rs_tma_kernel -c 1 -o gpurun_out/r02r/ncu_rs_default_c3 python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02r/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/r02r/ncu_rs_default_c3.ncu-rep --page details --csv > gpurun_out/r02r/ncu_rs_default_c3_details.csv 2>&1; wc -l gpurun_out/r02r/ncu_rs_default_c3_details.csv
