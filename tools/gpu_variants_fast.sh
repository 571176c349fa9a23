# usage: bash tools/gpu_variants_fast.sh "-DX=1" ...   rebuild per flag set on the box, then the
# bench's per-kernel times (no parity tests, no CPU baseline, no north-star block)
for v in "$@"; do
  touch paper_1503_03553_b200/csrc/*.cu
  make -C paper_1503_03553_b200 -j8 EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-north-star 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', 'value %.3e ms/step %.4f' % (d['value'], d['ms_per_step']), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
done
