#!/bin/bash
# One GPU call: the kernel bench, ncu --set full of every kernel at bench
# shapes summarised on the box (-> gpurun_out/ncu_traffic.json + a
# raw-metrics CSV; the .ncu-rep is deleted to stay under gpurun's 64 MiB
# pull limit), then the ncu launch list of one bench step.
mkdir -p gpurun_out
python -m paper_2305_18513_b200.kernel_bench > gpurun_out/kernel_bench.txt 2>&1
ncu --set full --clock-control none -o /tmp/kb_full -f \
    python -m paper_2305_18513_b200.kernel_bench --iters 1 --core > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/kb_full.ncu-rep gpurun_out/ncu_traffic.json > gpurun_out/ncu_summary.txt 2>&1
ncu -i /tmp/kb_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,launch__registers_per_thread,launch__grid_size,launch__block_size > gpurun_out/ncu_full_kernels.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-baseline-memory --no-cpu-baseline --no-kernel-timing \
    > gpurun_out/launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv gpurun_out/launches_summary.txt > /dev/null 2>&1
ls -la gpurun_out
