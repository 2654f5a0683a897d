# profiles/scripts/quick.sh TAG -- GPU-box quick look: bench (no CPU leg) + refine probe
mkdir -p gpurun_out/$1
timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err
timeout 120 python tests/refine_probe.py > gpurun_out/$1/probe.log 2>&1
cat gpurun_out/$1/probe.log
