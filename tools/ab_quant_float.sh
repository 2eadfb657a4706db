#!/bin/bash
# A/B: float vs integer quantiser on configs 4 and 2 (bench lines to gpurun_out/)
cd "$(dirname "$0")/.."  # repo root
mkdir -p gpurun_out/r2
for rep in 1 2; do
  for qf in 1 0; do
    ADCT_QUANT_FLOAT=$qf python bench.py --config 4 --steps 10 --warmup 5 --no-e2e --no-cpu > gpurun_out/r2/ab_qf${qf}_c4_$rep.json 2>/dev/null
    ADCT_QUANT_FLOAT=$qf python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/r2/ab_qf${qf}_c2_$rep.json 2>/dev/null
  done
done
for f in gpurun_out/r2/ab_qf*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['roofline']['kernel_ms'], d['clocks']['sm_mhz'], d['quant_jit'])"; done
