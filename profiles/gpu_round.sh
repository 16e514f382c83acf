set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python -m pytest tests -m gpu -q -x > gpurun_out/t3.log 2>&1; tail -8 gpurun_out/t3.log
python bench.py --steps 10 --warmup 3 > gpurun_out/b3.log 2>&1; tail -c 4000 gpurun_out/b3.log
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/b3ref.log 2>&1; tail -c 1500 gpurun_out/b3ref.log
