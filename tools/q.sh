timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bottom" 2>&1 | tail -3 > gpurun_out/q_test.txt
for bn in 128 64 0; do MG_BOTTOM_N=$bn timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_b$bn.log 2>&1; done
for bn in 128 0; do MG_BOTTOM_N=$bn timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 200 --n 256 > gpurun_out/bq_n256_b$bn.log 2>&1; done
