#!/bin/bash
# final check of the committed state: every GPU test (incl. the bench JSON test) and smoke
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final2_tests.log
tail -3 gpurun_out/final2_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
