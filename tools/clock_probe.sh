# bench.py step-time spread vs the clock sampler period (OTK_CLOCK_PERIOD, 0 = off)
mkdir -p gpurun_out
for rep in 1 2; do
for per in 0 0.01 0.05; do
  for k in 3 1; do
    OTK_CLOCK_PERIOD=$per python bench.py --config $k --no-cpu --no-e2e > gpurun_out/r14_cfg${k}_p${per}_$rep.json 2>&1
  done
done
done
for f in gpurun_out/r14_*.json; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', '%.4f ms/step'%d['ms_per_step'], d['run']['step_ms'], 'ttt %.3f'%d['run']['time_to_tolerance_ms'], d['clocks'].get('samples'), d['clocks'].get('sm_mhz'))
"; done
