# cfg5 bench with alternative libmapi builds (items per thread of the merge-path gather)
for v in base ipt12 ipt16; do
  if [ "$v" != base ]; then cp scripts/bin/libmapi_$v.so paper_2110_12065_b200/libmapi.so; fi
  timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_cfg5_$v.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg5_$v.log').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'])"
done
