# profiles/scripts/ab_so.sh -- GPU-box A/B of two builds of the product library (ab/A.so, ab/B.so), alternating bench runs
L=paper_2012_12544_b200/libbapipe_b200.so
cp $L ab/cur.so
for rep in 1 2 3; do
  for v in A B; do
    cp ab/$v.so $L
    timeout 300 python bench.py --no-cpu-baseline --no-per-call --steps 10 > /tmp/b_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('/tmp/b_$v.json'));k=d['kernels'];print('$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), {x: round(y,2) for x,y in k['phases_ms_per_step'].items()}, round(k['sim_flow64']['ms_per_step'],2), round(k['sim_flow32']['ms_per_step'],2))"
  done
done
cp ab/cur.so $L
