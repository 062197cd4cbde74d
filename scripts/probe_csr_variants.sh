# cfg5 bench with alternative libmapi builds: bash scripts/probe_csr_variants.sh t128 t512 ...
# ("default" = the in-tree build; others = scripts/bin/libmapi_<name>.so; default is re-run last)
mkdir -p gpurun_out
cp paper_2110_12065_b200/libmapi.so /tmp/libmapi_default.so
for v in default "$@" default; do
  if [ "$v" = default ]; then cp /tmp/libmapi_default.so paper_2110_12065_b200/libmapi.so;
  else cp scripts/bin/libmapi_$v.so paper_2110_12065_b200/libmapi.so; fi
  timeout 600 python bench.py --workload ${WORKLOAD:-cfg5} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_var_$v.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/bench_var_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), d['ms_per_step'], d['roofline'].get('kernel_ms_avg'))"
done
cp /tmp/libmapi_default.so paper_2110_12065_b200/libmapi.so
