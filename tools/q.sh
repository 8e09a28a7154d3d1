python bench.py > gpurun_out/bench_r01e.log 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python bench.py --config 4 --no-cpu-baseline --no-solve > gpurun_out/bench_c4.log 2>&1
python bench.py --config 2 --no-cpu-baseline --no-solve > gpurun_out/bench_c2.log 2>&1
python bench.py --config 1 --no-cpu-baseline --no-solve > gpurun_out/bench_c1.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01e.csv python tools/two_cycles.py > /dev/null 2>&1
