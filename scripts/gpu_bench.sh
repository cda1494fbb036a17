# quick perf iteration: build check + bench only (per-kernel table printed)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('value', round(d['value'],2), 'it/s  ms/step', round(d['ms_per_step'],2), 'iter-frac', round(d['iteration_roofline']['frac'],3), 'tts', round(d['time_to_solution']['ms'],2))
for k,v in d['kernels'].items(): print(f"  {k:15s} {v['avg_ms']:.3f} ms  {v['alg_GBps']:.0f} GB/s  x{v['launches']}")
print('clocks', d['clocks']); print('trisor', d.get('trisor')); print('e2e', d['e2e'])
PY
