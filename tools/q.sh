python -m pytest tests/test_gpu_parity.py -q -x -k "vanka_sweep or cycle_history or fused" 2>&1 | tail -2 > gpurun_out/q_test.txt
python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"march2_kernelILb0ELb0" -c 1 -o gpurun_out/prof_pl python tools/two_cycles.py > /dev/null 2>&1
