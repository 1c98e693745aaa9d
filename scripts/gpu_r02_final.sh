#!/bin/bash
# end-of-round evidence: GPU tests, smoke, the default bench line (c2) + reference arm, c3 line,
# and the ncu launch list of a short c2 run (each ncu pass only after its command exited 0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final_tests.log
tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err; echo "c2 rc=$?"
python bench.py --impl reference > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err; echo "ref rc=$?"
python bench.py --config c3 --no-cpu-baseline > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err; echo "c3 rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --max-new 32 --no-cpu-baseline --no-ar --no-profile"
$CMD > gpurun_out/final_prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv --log-file gpurun_out/final_launches_c2.csv $CMD > gpurun_out/final_ncu_launch.log 2>&1
echo "ncu rc=$?"
for f in final_bench_c2 final_reference final_bench_c3; do tail -c 400 gpurun_out/$f.json; echo; done
