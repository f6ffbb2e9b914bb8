mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/po_tests.log 2>&1; echo "rc $?" >> gpurun_out/po_tests.log
for cfg in bert-base-sst2 bert-base-sst2 bert-large-squad vit-b16-cifar100; do
python bench.py --config $cfg --no-cpu-baseline --no-baseline-memory > gpurun_out/ab.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg', round(d['ms_per_step'],2), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], {k:(round(v['avg_us'],1),round(v['frac'],3)) for k,v in d['kernels'].items() if 'attention_fwd' in k or 'gelu_fwd' in k})" >> gpurun_out/po_tests.log
done
grep -v "^\.\|^$" gpurun_out/po_tests.log | tail -8
