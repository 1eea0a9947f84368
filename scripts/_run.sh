timeout 300 python scripts/probe_single_phases.py 64 128 > gpurun_out/phases2.log 2>&1
timeout 300 python -m pytest tests/test_cascade_gpu.py tests/test_baseline_parity_gpu.py -k "query or serial or server or cascade" -q -p no:cacheprovider > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
timeout 600 python bench.py --no-stages --no-cpu --steps 10 > gpurun_out/b5.out 2> gpurun_out/b5.err
