python -m pytest tests/test_gpu_parity.py -q -x -k "fused or vanka_sweep" 2>&1 | tail -1 > gpurun_out/q_test.txt
for f in 1 0; do MG_FUSE_PROLONG=$f python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_$f.log 2>&1; done
