#!/bin/bash
# summarise bench JSON lines in gpurun_out/<tag>_*
for f in gpurun_out/$1*bench*.log; do echo "== $f"; grep '^{' $f | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); r=d.get('roofline') or {}; print(d['n_gpus'], d['config'].get('per_gpu_batch'), d['config'].get('exchange'), 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'eager', round(d.get('ms_per_step_eager',0),3), 'dom_ms', r.get('avg_launch_ms_in_step'), 'frac', r.get('frac'), 'nvl', (d.get('roofline_nvlink') or {}).get('achieved'), 'e2e', (d.get('e2e') or {}).get('value'), 'launches', d.get('gpu_launches'), 'clk', (d.get('clocks') or {}).get('sm_mhz'))
"; grep -iE "error|Traceback" $f | head -3; done
