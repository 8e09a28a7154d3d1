set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exact.py -x -q -k "bsr or exact" --durations=8 > gpurun_out/s3_bsr.log 2>&1; echo "rc=$?" >> gpurun_out/s3_bsr.log
timeout 300 python -m pytest tests/test_gpu_golden.py -x -q > gpurun_out/s3_gold.log 2>&1; echo "rc=$?" >> gpurun_out/s3_gold.log
for C in 2 4; do
B="python bench.py --config $C --relax bsr --no-cpu-baseline --no-e2e --no-solve"
timeout 200 $B > gpurun_out/s3_jf_c${C}_1.json 2> gpurun_out/s3_jf_c${C}_1.err
MG_JACOBI_FUSE_B=0 timeout 200 $B > gpurun_out/s3_jf_c${C}_0.json 2> gpurun_out/s3_jf_c${C}_0.err
done
