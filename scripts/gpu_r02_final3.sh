#!/bin/bash
# final state: every GPU test, smoke, the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final3_tests.log
tail -3 gpurun_out/final3_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/final3_bench_c2.json 2> gpurun_out/final3_bench_c2.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/final3_bench_c2.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['rollout']['frac'], d['host_loop'], d['clocks'])"
