# profiles/scripts/ab_parts.sh -- GPU-box A/B: 2 vs 3 concurrent parts (BP_SPLIT_PARTS), alternating bench runs
for rep in 1 2 3; do
  for n in 2 3; do
    BP_SPLIT_PARTS=$n timeout 300 python bench.py --no-cpu-baseline --no-per-call --steps 10 > /tmp/b_$n.json 2>/dev/null
    python -c "import json;d=json.load(open('/tmp/b_$n.json'));print('parts $n', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"
  done
done
BP_SPLIT_PARTS=3 timeout 300 python tests/timeline_probe.py | head -75
