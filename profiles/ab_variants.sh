#!/bin/bash
# A/B of K1 build variants (variants/lib<NAME>.so vs the main library): the
# bench's fused rollout+score kernel time and the step value, per workload.
# usage: bash profiles/ab_variants.sh "main W1 W2" "manipulator3 dubins"
LIBS=${1:-"main"}; WLS=${2:-"manipulator3 dubins aliengo_lipm"}
for rep in 1 2; do
for lib in $LIBS; do
  if [ $lib = main ]; then unset CACTO_B200_LIB; else export CACTO_B200_LIB=$PWD/variants/lib$lib.so; fi
  for w in $WLS; do python bench.py --steps 5 --warmup 3 --no-cpu --no-secondary --workload $w 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$lib $w\", round(d[\"value\"]/1e6,2), 'M/s  K1', round(d[\"roofline\"][\"kernel_ms\"],4), 'ms', round(d[\"roofline\"][\"frac\"],4))"; done
done
done
