# profiles/scripts/tl.sh TAG -- GPU-box: launch timeline of one C5 sweep (split on) + a short bench
mkdir -p gpurun_out/$1
timeout 300 python tests/timeline_probe.py > gpurun_out/$1/timeline.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-per-call --steps 5 > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err
cat gpurun_out/$1/timeline.txt
python -c "import json;d=json.load(open('gpurun_out/$1/bench.json'));print('device',d['ms_per_step'],'e2e',d['e2e']['ms_per_step'])"
