set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2s_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1
python bench.py > gpurun_out/r2s_bench_c5.json 2> gpurun_out/r2s_bench_c5.err
for C in 2 3 4; do python bench.py --config $C --no-cpu-baseline > gpurun_out/r2s_bench_c$C.json 2> gpurun_out/r2s_bench_c$C.err; done
python bench.py --config 4 --relax vanka --no-cpu-baseline > gpurun_out/r2s_bench_c4v.json 2> gpurun_out/r2s_bench_c4v.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2s_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-solve > gpurun_out/r2s_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vanka_warp|restrict_march|vanka_bnd2" -c 9 -o gpurun_out/r2s_full python tools/two_cycles.py > gpurun_out/r2s_ncu_full.log 2>&1
