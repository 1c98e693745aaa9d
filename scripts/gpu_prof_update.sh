#!/bin/bash
# kernel split of one online draft update at the c3/c4 shape (ncu launch list of the second update)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/prof_update.py c3 32 512 2 > gpurun_out/upd_plain.log 2>&1 || exit 1
cat gpurun_out/upd_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/upd_launches.csv \
    python scripts/prof_update.py c3 32 512 2 > gpurun_out/upd_ncu.log 2>&1
python scripts/ncu_summary.py list gpurun_out/upd_launches.csv > gpurun_out/upd_launches.txt 2>&1
head -30 gpurun_out/upd_launches.txt
