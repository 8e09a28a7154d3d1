MG_NVCC_EXTRA=-DMG_PROL_NOOP python paper_2107_04060_b200/build.py > /dev/null 2>&1
python bench.py --no-cpu-baseline --no-e2e --no-solve --steps 100 > gpurun_out/bq_noop.log 2>&1
