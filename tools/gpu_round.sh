# Round evidence on one GPU box: GPU tests, smoke, bench lines of every config, launch list, ncu captures.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2y_gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r2y_bench_c5.json 2> gpurun_out/r2y_bench_c5.err
for C in 1 2 3 4; do timeout 200 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2y_bench_c$C.json 2> gpurun_out/r2y_bench_c$C.err; done
timeout 200 python bench.py --config 2 --relax bsr --no-cpu-baseline > gpurun_out/r2y_bench_c2bsr.json 2> gpurun_out/r2y_bench_c2bsr.err
timeout 200 python bench.py --config 4 --relax vanka --no-cpu-baseline > gpurun_out/r2y_bench_c4v.json 2> gpurun_out/r2y_bench_c4v.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2y_bench_ref.json 2> gpurun_out/r2y_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2y_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-solve > gpurun_out/r2y_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vanka_warp|restrict_march|vanka_bnd2" -c 15 -o gpurun_out/r2y_full python tools/two_cycles.py > gpurun_out/r2y_ncu_full.log 2>&1
CFG=4 RELAX=vanka timeout 600 ncu --set full --import-source on --clock-control none -k regex:"vanka_hwarp|vanka_bnd2|prolong_planes" -c 8 -o gpurun_out/r2y_hwarp python tools/two_cycles.py > gpurun_out/r2y_ncu_hwarp.log 2>&1
