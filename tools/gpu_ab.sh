set -x
B="python bench.py --no-cpu-baseline --no-e2e --no-solve"
for v in 128 40 56 80 200; do
MG_WARP_TARGET=$v timeout 200 $B > gpurun_out/s3_wt_$v.json 2> gpurun_out/s3_wt_$v.err
done
