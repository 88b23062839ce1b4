mkdir -p gpurun_out
one() { timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 "$@" > gpurun_out/r6v.json 2>/dev/null; tail -1 gpurun_out/r6v.json | python -c "
import sys, json; d = json.loads(sys.stdin.read()); r = d['roofline']
print('$*', '%.4e' % d['value'], round(d['ms_per_step'], 2), 'frac', round(r['frac'], 3), d['clocks']['sm_mhz'], d['clocks']['reasons'], [round(v/1e6,1) for v in d['repeats']['values']])"; }
for rep in 1 2; do
one
one --l2-prefetch 2
one --dyn-pct 0
one --l2-prefetch 2 --dyn-pct 0
done
LFOAM_LIB=liblfoam_old.so one --config 2
one --config 2
LFOAM_LIB=liblfoam_old.so one --config 2
one --config 2
