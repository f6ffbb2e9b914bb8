mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_codecs_gpu.py -x -q -k "prune" > gpurun_out/prune_tests.log 2>&1; echo "rc $?" >> gpurun_out/prune_tests.log
timeout 300 python tools/prune_phases.py > gpurun_out/phases.txt 2>&1
timeout 300 python -m paper_2305_18513_b200.kernel_bench --core > gpurun_out/kb_core.txt 2>&1
tail -5 gpurun_out/prune_tests.log; cat gpurun_out/phases.txt; grep -i "prune\|restore" gpurun_out/kb_core.txt
