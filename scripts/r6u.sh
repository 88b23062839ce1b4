mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv
for rep in 1 2 3; do
  timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r6u_driverlike_$rep.json 2> gpurun_out/r6u_driverlike_$rep.err
  tail -1 gpurun_out/r6u_driverlike_$rep.json | python -c "
import sys, json; d = json.loads(sys.stdin.read()); r = d['roofline']
print('$rep', '%.4e' % d['value'], round(d['ms_per_step'], 2), 'frac', round(r['frac'], 3), 'dram_frac', r.get('dram_frac'), 'traffic', r.get('traffic'), d['clocks'], 'e2e %.3e' % d['e2e']['value'], [round(v/1e6,1) for v in d['repeats']['values']])"
done
