for t in 32 16 8; do MG_MARCH_SMALL=$t python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_s$t.log 2>&1; done
