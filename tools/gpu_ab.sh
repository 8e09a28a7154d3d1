set -x
B="python bench.py --config 4 --relax vanka --no-cpu-baseline --no-e2e --no-solve"
timeout 200 $B > gpurun_out/s3_hv_def.json 2> gpurun_out/s3_hv_def.err
timeout 300 python -m pytest tests/test_gpu_het_vanka.py -x -q --durations=5 > gpurun_out/s3_het.log 2>&1; echo "rc=$?" >> gpurun_out/s3_het.log
