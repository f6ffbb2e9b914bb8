mkdir -p gpurun_out
for cfg in bert-base-sst2 bert-large-squad; do
for env in "SLIMFIT_PRUNE_HINT=1" "SLIMFIT_PRUNE_HINT=0" "SLIMFIT_PRUNE_HINT=1" "SLIMFIT_PRUNE_HINT=0" "SLIMFIT_SIDE_STREAM=0"; do
  env $env python bench.py --config $cfg --no-cpu-baseline --no-kernel-timing --no-baseline-memory > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg','$env',round(d['ms_per_step'],2),round(d['value'],1),round(d['e2e']['value'],1),d['clocks']['sm_mhz'],d['clocks']['reasons'])"
done; done > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
