set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "fgmres or paper_regime or timestep or fullsize or krylov" --durations=5 > gpurun_out/s3_fg.log 2>&1; echo "rc=$?" >> gpurun_out/s3_fg.log
