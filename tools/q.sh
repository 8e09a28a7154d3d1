python -m pytest tests/test_gpu_parity.py -q -x -k "vanka_sweep or cycle_history or restrict or solve_matches or fgmres" 2>&1 | tail -2 > gpurun_out/q_test.txt
MG_SMALL_TILE_N=0 python -m pytest tests/test_gpu_parity.py -q -x -k "vanka_sweep or cycle_history" 2>&1 | tail -2 >> gpurun_out/q_test.txt
for n in 64 256; do for st in 0 128; do MG_SMALL_TILE_N=$st python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 200 --n $n > gpurun_out/bq_n${n}_$st.log 2>&1; done; done
for st in 0 64 128 256; do MG_SMALL_TILE_N=$st python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_st$st.log 2>&1; done
