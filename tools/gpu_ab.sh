set -x
CFG=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bsr_" -c 5 -o gpurun_out/s3_bsr2 python tools/two_cycles.py > gpurun_out/s3_ncu_bsr2.log 2>&1
