# usage: bash tools/gpu_variants.sh VAR v1 v2 ...   (runs the bench once per value of env VAR)
var=$1; shift
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | head -2
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', 'value %.3e ms/step %.4f' % (d['value'], d['ms_per_step']), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
done
