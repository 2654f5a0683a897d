# profiles/scripts/ab_refine_sms.sh -- GPU-box A/B: refine on exclusive SMs (BP_REFINE_SMS) vs shared, alternating runs
for rep in 1 2 3; do
  for n in 0 80 110; do
    BP_REFINE_SMS=$n timeout 300 python bench.py --no-cpu-baseline --no-per-call --steps 10 > /tmp/b_$n.json 2>/dev/null
    python -c "import json;d=json.load(open('/tmp/b_$n.json'));print('sms $n', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"
  done
done
