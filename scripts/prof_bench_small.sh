#!/bin/bash
# Launch list + full captures of the dominant kernels of bench.py (run under gpurun).
set -e
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu --e2e-queries 200 > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --e2e-queries 200 > gpurun_out/ncu_launch.log 2>&1
python scripts/prof_cascade.py serial > gpurun_out/plain_serial.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:single -s 12 -c 1 \
    -o gpurun_out/r01_single python scripts/prof_cascade.py serial > gpurun_out/ncu_single.log 2>&1
python scripts/prof_cascade.py batch 96 > gpurun_out/plain_batch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cascade3d_kernel -s 2 -c 1 \
    -o gpurun_out/r01_sweep python scripts/prof_cascade.py batch 96 > gpurun_out/ncu_sweep.log 2>&1
python scripts/prof_field.py > gpurun_out/plain_field.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"zpass|fft_kernel" -s 8 -c 3 \
    -o gpurun_out/r01_field python scripts/prof_field.py > gpurun_out/ncu_field.log 2>&1
echo done
