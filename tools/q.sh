python -m pytest tests/ -q -x -m gpu 2>&1 | tail -2 > gpurun_out/q_test.txt
python bench.py > gpurun_out/bench_r01d.log 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python bench.py --config 4 --no-cpu-baseline --no-solve > gpurun_out/bench_c4.log 2>&1
python bench.py --config 2 --no-cpu-baseline --no-solve > gpurun_out/bench_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01d.csv python tools/two_cycles.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"march2_kernelILb0ELb0|restrict_march_kernelILb0" -c 2 -o gpurun_out/prof_r01d python tools/two_cycles.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"march2_kernelILb0ELb1" --launch-skip 3 -c 1 -o gpurun_out/prof_r01d_post python tools/two_cycles.py > /dev/null 2>&1
CFG=4 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"bsr_._march" -c 2 -o gpurun_out/prof_r01d_bsr python tools/two_cycles.py > /dev/null 2>&1
