mkdir -p gpurun_out/cap
for c in 0 16 8 4; do
  echo "== per_sm cap $c"
  BP_REFINE_PER_SM=$c timeout 300 python tests/timeline_probe.py > gpurun_out/cap/tl_$c.txt 2>&1
  head -1 gpurun_out/cap/tl_$c.txt; grep -E " refine | phase_refine" gpurun_out/cap/tl_$c.txt
  BP_REFINE_PER_SM=$c timeout 300 python tests/timeline_probe.py --no-split > gpurun_out/cap/tln_$c.txt 2>&1
  head -1 gpurun_out/cap/tln_$c.txt; grep -E " refine | phase_refine" gpurun_out/cap/tln_$c.txt
done
