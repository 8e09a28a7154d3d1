set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bsr" > gpurun_out/s3_bsr.log 2>&1; echo "rc=$?" >> gpurun_out/s3_bsr.log
timeout 600 python -m pytest tests/test_gpu_golden.py -x -q > gpurun_out/s3_gold.log 2>&1; echo "rc=$?" >> gpurun_out/s3_gold.log
B="python bench.py --config 4 --no-cpu-baseline --no-e2e --no-solve"
timeout 200 $B > gpurun_out/s3_c4_jp1.json 2> gpurun_out/s3_c4_jp1.err
MG_JACOBI_PAIR=0 timeout 200 $B > gpurun_out/s3_c4_jp0.json 2> gpurun_out/s3_c4_jp0.err
B="python bench.py --config 2 --relax bsr --no-cpu-baseline --no-e2e --no-solve"
timeout 200 $B > gpurun_out/s3_c2_jp1.json 2> gpurun_out/s3_c2_jp1.err
MG_JACOBI_PAIR=0 timeout 200 $B > gpurun_out/s3_c2_jp0.json 2> gpurun_out/s3_c2_jp0.err
