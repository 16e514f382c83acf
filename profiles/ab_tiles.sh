#!/bin/bash
# K1 time vs tiles in flight per SM (CACTO_ROLLOUT_TC_TILES = 1 / 2 / 4)
for t in 4 2 1; do
  for w in manipulator3 dubins; do
    CACTO_ROLLOUT_TC_TILES=$t python bench.py --steps 3 --warmup 2 --no-cpu --no-secondary --workload $w 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"tiles=$t $w\", round(d[\"value\"]/1e6,2), 'M/s  K1', round(d[\"roofline\"][\"kernel_ms\"],4), 'ms')"
  done
done
