mkdir -p gpurun_out
timeout 300 python tools/prune_phases.py > gpurun_out/phases.txt 2>&1
cat gpurun_out/phases.txt
