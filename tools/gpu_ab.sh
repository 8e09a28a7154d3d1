# session A/B: het warp sweep + plane-split prolongation
set -x
timeout 600 python -m pytest tests/test_gpu_het_vanka.py -x -q > gpurun_out/s3_het.log 2>&1; echo "rc=$?" >> gpurun_out/s3_het.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prolong or restrict" > gpurun_out/s3_prol.log 2>&1; echo "rc=$?" >> gpurun_out/s3_prol.log
timeout 200 python bench.py --config 4 --relax vanka --no-cpu-baseline --no-e2e --no-solve > gpurun_out/s3_c4v.json 2> gpurun_out/s3_c4v.err
MG_HET_WARP_N=0 timeout 200 python bench.py --config 4 --relax vanka --no-cpu-baseline --no-e2e --no-solve > gpurun_out/s3_c4v_off.json 2> gpurun_out/s3_c4v_off.err
timeout 200 python bench.py --config 4 --no-cpu-baseline --no-e2e --no-solve > gpurun_out/s3_c4.json 2> gpurun_out/s3_c4.err
MG_PROL_PLANES_N=0 timeout 200 python bench.py --config 4 --no-cpu-baseline --no-e2e --no-solve > gpurun_out/s3_c4_off.json 2> gpurun_out/s3_c4_off.err
timeout 600 python -m pytest tests/test_gpu_golden.py -x -q -k "4" > gpurun_out/s3_gold4.log 2>&1; echo "rc=$?" >> gpurun_out/s3_gold4.log
