# Config 2's block methods, one short bench run each; prints per-kernel fractions.
#   bash scripts/cfg2_methods.sh [steps]
STEPS=${1:-5}
for m in bl_bicg bl_bicg_rq bl_bicgstab_rq bl_qmr bl_bicgstab; do
  python bench.py --config 2 --method $m --steps $STEPS --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read())
ks = [(k['kernel'], k['frac'] and round(k['frac'], 3), round(k['share_of_step'], 3)) for k in d['iteration']['kernels']]
print('$m', round(d['value']), round(d['ms_per_step'], 3), round(d['iteration']['frac_of_peak'], 3), ks)"
done
