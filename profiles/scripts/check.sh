# profiles/scripts/check.sh TAG -- GPU-box check: smoke, pytest -m gpu, bench (no CPU leg), refine probe
mkdir -p gpurun_out/$1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$1/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$1/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err
timeout 120 python tests/refine_probe.py > gpurun_out/$1/probe.log 2>&1
tail -3 gpurun_out/$1/pytest_gpu.log
