# profiles/scripts/excl_probe.sh -- GPU-box: refine on exclusive SMs (BP_REFINE_SMS / BP_REFINE_WARPS) vs shared
for cfg in "0 8" "40 8" "60 8" "80 8" "60 4" "100 4"; do
  set -- $cfg
  echo "== BP_REFINE_SMS=$1 BP_REFINE_WARPS=$2"
  BP_REFINE_SMS=$1 BP_REFINE_WARPS=$2 timeout 300 python tests/timeline_probe.py | grep -E "split=| refine |minmax_dp_coarse|steps  3255"
  BP_REFINE_SMS=$1 BP_REFINE_WARPS=$2 timeout 300 python tests/timeline_probe.py --no-split | grep -E "split=| refine |minmax_dp_coarse|steps  3255"
done
