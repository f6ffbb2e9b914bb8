mkdir -p gpurun_out
timeout 300 python -m paper_2305_18513_b200.kernel_bench --core 2>&1 | grep layernorm_bwd > gpurun_out/lnb.txt
timeout 600 python -m pytest tests -q -x -m gpu -k "layernorm or ln_ or model or fused or wide or gemm" >> gpurun_out/lnb.txt 2>&1
python bench.py --config bert-base-sst2 --no-cpu-baseline --no-baseline-memory > gpurun_out/ab.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), {k:round(v['avg_us'],1) for k,v in d['kernels'].items() if 'layernorm_bwd' in k})" >> gpurun_out/lnb.txt
cat gpurun_out/lnb.txt | grep -v "^\.\|^$" | tail -8
