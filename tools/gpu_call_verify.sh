mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -m paper_2305_18513_b200.kernel_bench > gpurun_out/kernel_bench.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_prune -c 2 -o gpurun_out/prune -f python -m paper_2305_18513_b200.kernel_bench --iters 1 --core > gpurun_out/ncu_prune.log 2>&1
tail -3 gpurun_out/gpu_tests.log
