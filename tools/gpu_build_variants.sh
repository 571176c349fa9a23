# usage: bash tools/gpu_build_variants.sh "-DX=1" "-DX=2" ...  rebuilds the library per flag set on
# the box and runs the bench once per variant (parity tests run on the first variant)
first=1
for v in "$@"; do
  touch paper_1503_03553_b200/csrc/*.cu paper_1503_03553_b200/csrc/*.cpp
  make -C paper_1503_03553_b200 -j8 EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  if [ $first = 1 ]; then timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 | head -1; first=0; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', 'value %.3e ms/step %.4f' % (d['value'], d['ms_per_step']), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
done
