# round-2 final captures: bench launch list (headline), full capture of one serial-loop lone query
# (warm L2, ring + one CTA per SM), density kernels at the C5 bolt scale (128^3), the 512^3 landscape
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-stages --no-cpu --e2e-queries 200 > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --cache-control none --import-source on -k regex:cascade3d_single -s 3500 -c 1 -o gpurun_out/r02_single64_final python bench.py --steps 2 --warmup 3 --no-stages --no-cpu --e2e-queries 100 > gpurun_out/ncu_single.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|dist_wind_culled" -c 2 -o gpurun_out/r02_density_final python scripts/prof_density.py bolt_nut 128 > gpurun_out/ncu_dens.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"product_brick|fft_rows|fft_cols" -s 8 -c 4 -o gpurun_out/r02_field512_final python scripts/prof_field.py > gpurun_out/ncu_field.log 2>&1
