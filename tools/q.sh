python -m pytest tests/test_gpu_parity.py -q -x -k "cycle_history or fused" 2>&1 | tail -1 > gpurun_out/q_test.txt
python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_1.log 2>&1
