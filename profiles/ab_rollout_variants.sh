for lib in main D main D; do
  if [ $lib = D ]; then export CACTO_B200_LIB=$PWD/variants/libD.so; else unset CACTO_B200_LIB; fi
  for w in dubins manipulator3 aliengo_lipm; do python bench.py --steps 5 --warmup 3 --no-cpu --no-secondary --workload $w 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$lib $w\", round(d[\"value\"]/1e6,2), round(d[\"roofline\"][\"kernel_ms\"],4))"; done
done
