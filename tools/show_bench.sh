#!/bin/bash
for f in gpurun_out/bench_*.log; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print('$f'.split('/')[-1], round(d['value'],2), round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phases_ms_per_step'].items()}, r['kernel'], round(r['frac'],3), {k:round(v['frac'],3) for k,v in r['others'].items()})" 2>/dev/null || tail -3 $f; done
