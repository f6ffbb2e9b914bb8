python -m pytest tests/test_codecs_gpu.py tests/test_model_gpu.py -x -q -m gpu 2>&1 | tail -2
python -m paper_2305_18513_b200.kernel_bench > gpurun_out/kb.txt 2>&1
ncu --set full --clock-control none -k regex:k_p[123] -c 5 -o gpurun_out/p python -m paper_2305_18513_b200.kernel_bench --iters 1 > /dev/null 2>&1
grep prune gpurun_out/kb.txt
