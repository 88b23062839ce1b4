mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
for rep in 1 2; do
for dp in 0 25; do
  timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline --dyn-pct $dp > gpurun_out/r6q_c3_d${dp}_$rep.json 2>&1
  summ gpurun_out/r6q_c3_d${dp}_$rep.json "c3 dyn$dp"
  timeout 300 python bench.py --config 5 --renumber 1 --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline --dyn-pct $dp > gpurun_out/r6q_c5r_d${dp}_$rep.json 2>&1
  summ gpurun_out/r6q_c5r_d${dp}_$rep.json "c5rcm dyn$dp"
done
done
for dp in 0 25; do
  timeout 600 python bench.py --config 5 --renumber 0 --steps 4 --warmup 3 --repeats 2 --no-cpu-baseline --dyn-pct $dp > gpurun_out/r6q_c5_d${dp}.json 2>&1
  summ gpurun_out/r6q_c5_d${dp}.json "c5raw dyn$dp"
done
