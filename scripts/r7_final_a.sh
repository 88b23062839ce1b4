mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r7f_gpu_tests.log 2>&1; tail -3 gpurun_out/r7f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r7f_smoke.log 2>&1; tail -2 gpurun_out/r7f_smoke.log
bash scripts/bench_final.sh r7 > gpurun_out/r7f_bench.log 2>&1
grep -h '"metric"' gpurun_out/bench_r7_*.json | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d.get('roofline') or {}
    print(d['config'].get('workload'), d.get('impl'), '%.3e' % d['value'], 'ms/step', round(d.get('ms_per_step') or 0, 2), 'frac', r.get('frac'), d.get('clocks', {}).get('sm_mhz'), d.get('clocks', {}).get('reasons'))
"
