set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bsr" > gpurun_out/s3_bsr.log 2>&1; echo "rc=$?" >> gpurun_out/s3_bsr.log
B="python bench.py --config 4 --no-cpu-baseline --no-e2e --no-solve"
timeout 200 $B > gpurun_out/s3_c4_pre.json 2> gpurun_out/s3_c4_pre.err
timeout 200 $B > gpurun_out/s3_c4_pre2.json 2> gpurun_out/s3_c4_pre2.err
