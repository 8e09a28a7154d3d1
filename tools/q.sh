python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "fgmres or solve" 2>&1 | tail -2 > gpurun_out/q_test.txt
python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bq_solve5.log 2>&1
MG_CGS_PASSES=1 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bq_solve5_1.log 2>&1
python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bq_solve3.log 2>&1
