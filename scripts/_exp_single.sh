timeout 120 python scripts/probe_e2e.py 64 2>&1 | grep -E "^B|^D|^F"
timeout 300 python -m pytest tests/test_cascade_gpu.py tests/test_haptic_gpu.py tests/test_energy_gpu.py -x -q 2>&1 | tail -1
timeout 120 python scripts/probe_single_phases.py 8 64 | head -16
