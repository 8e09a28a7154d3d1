python -m pytest tests/test_gpu_parity.py -q -x -k "bsr" 2>&1 | tail -2 > gpurun_out/q_test.txt
python bench.py --config 4 --no-cpu-baseline --no-e2e --no-solve --steps 50 > gpurun_out/bq_c4.log 2>&1
