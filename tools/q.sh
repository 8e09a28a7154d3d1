for rm in 512 100000 512; do MG_RESID_MARCH_N=$rm python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bq_rm$rm.log 2>&1; tail -1 gpurun_out/bq_rm$rm.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($rm, round(d['ms_per_step'],3), d['solve']['iterations'], round(d['solve']['ms'],1))" >> gpurun_out/rm.txt; done
