mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
timeout 900 python -m pytest tests/test_gpu_hbm.py -q -x -k "runtime" > gpurun_out/r6s_tests.log 2>&1; tail -1 gpurun_out/r6s_tests.log
for rep in 1 2; do
for dp in 0 25 33 40 50; do
  timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline --dyn-pct $dp > gpurun_out/r6s_c3_d${dp}_$rep.json 2>&1
  summ gpurun_out/r6s_c3_d${dp}_$rep.json "c3 dyn$dp"
done
done
