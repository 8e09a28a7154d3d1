for ps in 1 2 3; do MG_PROL_SEG=$ps python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_ps$ps.log 2>&1; done
