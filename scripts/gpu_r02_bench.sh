#!/bin/bash
# round-2 bench lines (c2 default, c3) + the c2 launch list + tcgen05 tensor-pipe activity of the GEMMs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
tail -c 300 gpurun_out/r02_bench_c2.json
python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
tail -c 300 gpurun_out/r02_bench_c3.json
SHORT="python bench.py --steps 1 --warmup 0 --max-new 24 --no-cpu-baseline --no-ar --no-profile"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file gpurun_out/r02_launches_c2.csv $SHORT > gpurun_out/r02_ncu_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:gemm -s 600 -c 40 --csv --log-file gpurun_out/r02_gemm_tensor_c2.csv $SHORT > gpurun_out/r02_ncu_gemm.log 2>&1
ls -la gpurun_out | tail -5
