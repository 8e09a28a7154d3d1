python -m pytest tests/test_gpu_parity.py -q -x -k "cycle_history" 2>&1 | tail -3 > gpurun_out/q_test.txt
