python -m pytest tests/test_gpu_parity.py -q -x -k "fused or cycle_history or fgmres or solve_matches" 2>&1 | tail -2 > gpurun_out/q_test.txt
for f in 1 0; do MG_FUSE_PROLONG=$f python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_f$f.log 2>&1; done
for f in 1 0; do MG_FUSE_PROLONG=$f python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 200 --config 2 > gpurun_out/bq_c2_f$f.log 2>&1; done
