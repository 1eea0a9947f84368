#!/bin/bash
# Launch list of bench.py's timed kernels (run under gpurun; ONE ncu pass).
# Full captures of individual kernels are separate gpurun calls:
#   ncu --set full --cache-control none --clock-control none --import-source on -k regex:single -s 25 -c 1 \
#       -o gpurun_out/X python scripts/prof_single_small.py 64
#   ... -k regex:cascade3d_kernel -s 2 -c 1 ... python scripts/prof_cascade.py batch 96
#   ... -k regex:"product_brick|fft_rows_staged|fft_cols_tma" -c 3 ... python scripts/prof_field.py
set -e
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu --no-stages --e2e-queries 200 > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-stages --e2e-queries 200 > gpurun_out/ncu_launch.log 2>&1
echo done
