set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python -m pytest tests -m gpu -q > gpurun_out/tests.log 2>&1; tail -15 gpurun_out/tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 5000 gpurun_out/bench.log
