set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python -m pytest tests -m gpu -q > gpurun_out/tests.log 2>&1; tail -5 gpurun_out/tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 7000 gpurun_out/bench.log
python profiles/parity_probe.py > gpurun_out/probe.json 2> gpurun_out/probe.err; tail -2 gpurun_out/probe.err
