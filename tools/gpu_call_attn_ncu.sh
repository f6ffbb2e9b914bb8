mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_attn_fwd_tc5h -c 1 -o gpurun_out/attnf -f python -m paper_2305_18513_b200.kernel_bench --iters 1 --core > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out/attnf.ncu-rep
