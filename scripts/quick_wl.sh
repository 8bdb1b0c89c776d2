#!/bin/bash
# quick check of the warp-line path on a GPU box: parity vs the generic path,
# the C1/C3 tests, and the C3 bench line (no other legs)
python scripts/ab_wl_iter.py 2>&1 | tail -6
python -m pytest tests/test_gpu_fast.py -x -q -s 2>&1 | grep -E "C3 fp32|passed|failed|Error" | head
python bench.py --steps 5 --warmup 3 --no-ospr --no-search --no-c5 --no-c6 --no-e2e --no-fp64 > gpurun_out/quick.json 2> gpurun_out/quick.err
python -c "
import json;d=json.loads(open('gpurun_out/quick.json').read().strip().splitlines()[-1]);r=d['roofline']
print('it/s', round(d['value']), 'frac', round(r['frac'],4), 'per-iter', round(r['per_iteration']['ms']*1000,2), 'us', round(r['per_iteration']['frac'],4))"
