#!/bin/bash
# decode-step costs (prefill excluded) and per-class split: c3r at B = 4 / 16, c5 at B = 48 over a 2k context
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/bench_lowb.py 4 16 --config=c3r > gpurun_out/r02_step_costs_c3r.jsonl 2>&1
timeout 900 python scripts/bench_lowb.py 48 --config=c5 --ctx=2048 > gpurun_out/r02_step_costs_c5.jsonl 2>&1
cat gpurun_out/r02_step_costs_c3r.jsonl gpurun_out/r02_step_costs_c5.jsonl
