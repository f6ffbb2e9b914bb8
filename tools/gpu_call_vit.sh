mkdir -p gpurun_out
for env in "SLIMFIT_PLANES_ONLY=1" "SLIMFIT_PLANES_ONLY=0" "SLIMFIT_PLANES_ONLY=1" "SLIMFIT_PLANES_ONLY=0"; do
  env $env python bench.py --config vit-b16-cifar100 --no-cpu-baseline --no-kernel-timing --no-baseline-memory > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$env',round(d['ms_per_step'],2),round(d['e2e']['value'],1),d['step_ms'][:3],d['clocks']['sm_mhz'])"
done > gpurun_out/vit_ab.txt 2>&1
cat gpurun_out/vit_ab.txt
