mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
timeout 900 python -m pytest tests/test_gpu_dic.py -q -x > gpurun_out/r6l_tests.log 2>&1; tail -2 gpurun_out/r6l_tests.log
for rep in 1 2; do
for pf in 1 2; do
  timeout 300 python bench.py --precond DIC --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline --l2-prefetch $pf > gpurun_out/r6l_dic_pf${pf}_$rep.json 2>&1
  summ gpurun_out/r6l_dic_pf${pf}_$rep.json "c3 DIC pf$pf"
done
done
for pf in 1 2; do
  timeout 600 python bench.py --precond DIC --config 4 --steps 3 --warmup 3 --repeats 2 --no-cpu-baseline --l2-prefetch $pf > gpurun_out/r6l_dic4_pf${pf}.json 2>&1
  summ gpurun_out/r6l_dic4_pf${pf}.json "c4 DIC pf$pf"
done
