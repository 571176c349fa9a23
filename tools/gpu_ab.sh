# quick A/B: parity tests + bench at 262K + sweep at 8M
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | head -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('262K value %.3e ms/step %.4f' % (d['value'], d['ms_per_step']), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
rm -f gpurun_out/sweep.jsonl; timeout 600 python tools/scale_sweep.py ${SWEEP:-c4_8m} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['case'], 'ms/step %.3f PU/s %.3g' % (d['ms_per_step'], d['pu_s']), d['kernel_ms'])"
