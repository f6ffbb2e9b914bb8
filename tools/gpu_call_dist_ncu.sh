mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_dist_chunks -c 40 -o gpurun_out/dist -f python -m paper_2305_18513_b200.kernel_bench --iters 1 > gpurun_out/ncu_dist.log 2>&1
ls -la gpurun_out/dist.ncu-rep; tail -3 gpurun_out/ncu_dist.log
