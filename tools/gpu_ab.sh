set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_exact.py tests/test_gpu_api.py -x -q -k "bsr or golden or exact or api" > gpurun_out/s3_bsr.log 2>&1; echo "rc=$?" >> gpurun_out/s3_bsr.log
for C in 2 4; do
B="python bench.py --config $C --relax bsr --no-cpu-baseline --no-e2e --no-solve"
timeout 200 $B > gpurun_out/s3_pf_c${C}.json 2> gpurun_out/s3_pf_c${C}.err
done
