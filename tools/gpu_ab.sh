set -x
for C in 2 3; do
B="python bench.py --config $C --no-cpu-baseline --no-e2e --no-solve"
timeout 200 $B > gpurun_out/s3_t_c${C}_def.json 2> gpurun_out/s3_t_c${C}_def.err
MG_SMALL_TILE_N=256 timeout 200 $B > gpurun_out/s3_t_c${C}_256.json 2> gpurun_out/s3_t_c${C}_256.err
done
timeout 300 python -m pytest tests/test_gpu_golden.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s3_gold.log 2>&1; echo "rc=$?" >> gpurun_out/s3_gold.log
