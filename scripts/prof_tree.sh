#!/bin/bash
# tree_attn_kernel: microbenchmark + one ncu --set full capture per shape (B=1 x 211 rows, B=48 x 4 rows)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/bench_tree_attn2.py > gpurun_out/tree_attn.jsonl 2>&1
cat > /tmp/one_tree.py <<'PY'
import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2509_21792_b200 import capi
B, N, ctx, H = (int(x) for x in sys.argv[1:5])
t = C.c_double()
capi.dev_lib().sgb_bench_tree_attention_tree(B, N, ctx, H, 128, 3, C.byref(t))
print(t.value)
PY
for shape in "1 211 640 28" "48 4 2200 32"; do
  tag=$(echo $shape | tr ' ' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 2 -c 1 \
      -o gpurun_out/tree_$tag python /tmp/one_tree.py $shape > gpurun_out/ncu_tree_$tag.log 2>&1
done
ls -la gpurun_out
