mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --config vit-b16-cifar100 > gpurun_out/bench_vit.json 2> gpurun_out/bench_vit.err
python bench.py --config bert-large-squad > gpurun_out/bench_bl.json 2> gpurun_out/bench_bl.err
python -m paper_2305_18513_b200.kernel_bench > gpurun_out/kernel_bench.txt 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log
