mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_codecs_gpu.py -x -q -k "pack or quant4 or gelu or codec" > gpurun_out/pack_tests.log 2>&1; echo "rc $?" >> gpurun_out/pack_tests.log
timeout 300 python -m paper_2305_18513_b200.kernel_bench --core > gpurun_out/kb_core.txt 2>&1
tail -3 gpurun_out/pack_tests.log; grep -i "pack\|quant" gpurun_out/kb_core.txt
