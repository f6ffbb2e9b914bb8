mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_codecs_gpu.py -x -q -k "prune" > gpurun_out/prune_tests.log 2>&1; echo "rc $?" >> gpurun_out/prune_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/prune_tests.log
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'],d['clocks'])"
