mkdir -p gpurun_out
for v in 1 0; do echo "pf $v"; SLIMFIT_LNB_PF=$v timeout 300 python -m paper_2305_18513_b200.kernel_bench --core 2>&1 | grep layernorm_bwd_sparse; done > gpurun_out/lnb.txt 2>&1
for v in 4 3; do echo "pf 1 per_sm $v"; SLIMFIT_LNB_PER_SM=$v timeout 300 python -m paper_2305_18513_b200.kernel_bench --core 2>&1 | grep layernorm_bwd_sparse; done >> gpurun_out/lnb.txt 2>&1
timeout 600 python -m pytest tests -q -x -m gpu -k "layernorm or ln_ or model or fused" >> gpurun_out/lnb.txt 2>&1
cat gpurun_out/lnb.txt | tail -15
