#!/bin/bash
# A/B of an environment switch: bash profiles/ab_env.sh VAR "v1 v2" "workloads"
VAR=$1; VALS=$2; WLS=${3:-"manipulator3 dubins"}
for rep in 1 2; do for v in $VALS; do for w in $WLS; do
  env $VAR=$v python bench.py --steps 5 --warmup 3 --no-cpu --no-secondary --workload $w 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$VAR=$v $w\", round(d[\"value\"]/1e6,2), 'M/s  e2e', round(d[\"e2e\"][\"value\"]/1e6,2), ' K1', round(d[\"roofline\"][\"kernel_ms\"],4), 'ms  step', round(d[\"ms_per_step\"],4))"
done; done; done
