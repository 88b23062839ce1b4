mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r7_driverlike_$rep.json 2> gpurun_out/r7_driverlike_$rep.err
  tail -1 gpurun_out/r7_driverlike_$rep.json | python -c "
import sys, json; d = json.loads(sys.stdin.read()); r = d['roofline']
print('$rep', '%.4e' % d['value'], round(d['ms_per_step'], 2), 'frac', round(r['frac'], 3), 'dram_frac', round(r.get('dram_frac') or 0, 3), 'traffic', r.get('traffic'), d['clocks'], 'e2e %.3e' % d['e2e']['value'], 'launches', d['gpu_launches'])"
done
