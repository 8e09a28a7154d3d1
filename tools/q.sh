python -m pytest tests/test_gpu_parity.py -q -x -k "vanka_sweep or cycle_history or residual or bsr_sweep or fused" 2>&1 | tail -2 > gpurun_out/q_test.txt
python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_1.log 2>&1
python bench.py --config 4 --no-cpu-baseline --no-e2e --no-solve --steps 50 > gpurun_out/bq_c4.log 2>&1
