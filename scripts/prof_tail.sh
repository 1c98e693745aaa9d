#!/bin/bash
# Low-concurrency, HBM-bound tail at the 7B shape (c3, B = 1, AR steps): GEMM streaming rate at
# M = 1 per weight, the per-step device time (A/B: SGB_L2_PF_MB=0 turns the GEMM's pre-wait L2
# weight prefetch off), and an ncu launch list with per-launch DRAM bytes (the achieved GB/s of
# every kernel of a decode step). ncu runs only after the plain run exited 0.
mkdir -p gpurun_out
G="1x10752x3584 1x3584x3584 1x18944x3584 1x3584x18944 1x152064x3584 16x10752x3584 16x3584x18944"
for pf in 0 48; do
  echo "== SGB_L2_PF_MB=$pf"
  SGB_L2_PF_MB=$pf timeout 300 python scripts/bench_gemm.py $G 2>&1
  SGB_L2_PF_MB=$pf timeout 600 python scripts/bench_lowb.py 1 4 16 --config=c3 --vanilla 2>&1 || exit 1
done > gpurun_out/tail_ab.log
cat gpurun_out/tail_ab.log
timeout 300 python scripts/bench_lowb.py 1 --config=c3 --vanilla --ncu > /dev/null 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/tail_launches.csv python scripts/bench_lowb.py 1 --config=c3 --vanilla --ncu > gpurun_out/tail_ncu.log 2>&1
echo ncu=$?; wc -l gpurun_out/tail_launches.csv
