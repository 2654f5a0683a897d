# profiles/scripts/round.sh TAG -- the GPU-box command behind a round's profiles/:
# smoke, pytest -m gpu, bench (both arms), the refine walk micro-benchmark, the
# ncu launch list of bench.py, and one ncu --set full capture of the top kernels.
TAG=${1:-run}
set -x
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$TAG/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/$TAG/bench_reference.json 2> gpurun_out/$TAG/bench_ref.err
timeout 120 ./tests/cpp/refine_walk_bench tests/cpp/refine_q18895.bin > gpurun_out/$TAG/refine_walk.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-call > gpurun_out/$TAG/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sim_exact|k_sim_flow|k_refine_fast|k_partition|k_prune$" -c 8 -o gpurun_out/$TAG/full python tests/prof_sweep.py > gpurun_out/$TAG/ncu_full.log 2>&1
ls -la gpurun_out/$TAG
