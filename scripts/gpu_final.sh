#!/bin/bash
# End-of-session check: the driver's round-end sequence (GPU tests, smoke, default bench, reference
# arm), the B = 1 tail launch list after this session's kernel changes, and the c4 line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_gpu.log 2>&1; tail -3 gpurun_out/f_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/f_bench.log 2>&1; grep '^{' gpurun_out/f_bench.log | tail -1 | cut -c1-160
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.log 2>&1; grep '^{' gpurun_out/f_ref.log | tail -1 | cut -c1-160
timeout 300 python scripts/bench_lowb.py 1 --config=c3 --vanilla --ncu > /dev/null 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/f_tail_launches.csv python scripts/bench_lowb.py 1 --config=c3 --vanilla --ncu > gpurun_out/f_tail_ncu.log 2>&1; echo ncu=$?
timeout 1200 python bench.py --config c4 --no-cpu-baseline > gpurun_out/f_bench_c4.log 2>&1; grep '^{' gpurun_out/f_bench_c4.log | tail -1 | cut -c1-160
