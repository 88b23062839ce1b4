mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
timeout 900 python -m pytest tests/test_gpu_dic.py -q -x > gpurun_out/r6w_tests.log 2>&1; tail -1 gpurun_out/r6w_tests.log
for rep in 1 2; do
for dp in 0 30 50; do
  timeout 300 python bench.py --precond DIC --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline --dyn-pct $dp > gpurun_out/r6w_d${dp}_$rep.json 2>&1
  summ gpurun_out/r6w_d${dp}_$rep.json "c3 DIC dyn$dp"
done
done
for dp in 0 30; do
  timeout 600 python bench.py --precond DIC --config 4 --steps 3 --warmup 3 --repeats 2 --no-cpu-baseline --dyn-pct $dp > gpurun_out/r6w_c4_d$dp.json 2>&1
  summ gpurun_out/r6w_c4_d$dp.json "c4 DIC dyn$dp"
done
