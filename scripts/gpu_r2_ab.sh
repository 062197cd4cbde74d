mkdir -p gpurun_out
run() { # dir tag
  (cd $1 && MAPI_PLAN_TRACE=1 timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2> $GRAFT_REPO_ROOT/gpurun_out/ab_$2.err > $GRAFT_REPO_ROOT/gpurun_out/ab_$2.json; grep "plan trace" $GRAFT_REPO_ROOT/gpurun_out/ab_$2.err | tail -2; python -c "
import json; d=json.loads(open('$GRAFT_REPO_ROOT/gpurun_out/ab_$2.json').read().strip().splitlines()[-1]); print('$2', d['value'], d['roofline']['frac'])")
}
run _old old1
run . new1
run _old old2
run . new2
