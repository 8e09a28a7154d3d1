python -m pytest tests/ -q -x -m gpu 2>&1 | tail -2 > gpurun_out/q_test.txt
python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_1.log 2>&1
python bench.py --config 4 --no-cpu-baseline --no-e2e --no-solve --steps 50 > gpurun_out/bq_c4.log 2>&1
