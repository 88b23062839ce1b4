mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
timeout 900 python -m pytest tests/test_gpu_hbm.py tests/test_gpu_parity.py -q -x > gpurun_out/r6c_tests.log 2>&1; tail -2 gpurun_out/r6c_tests.log
for pf in 0 2 0 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline --l2-prefetch $pf > gpurun_out/r6c_c3_pf$pf.json 2>&1
  summ gpurun_out/r6c_c3_pf$pf.json "c3 pf$pf"
done
for pf in 0 2; do
  timeout 300 python bench.py --config 5 --renumber 1 --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline --l2-prefetch $pf > gpurun_out/r6c_c5r_pf$pf.json 2>&1
  summ gpurun_out/r6c_c5r_pf$pf.json "c5rcm pf$pf"
done
timeout 600 python bench.py --config 4 --steps 4 --warmup 3 --repeats 2 --no-cpu-baseline > gpurun_out/r6c_c4.json 2>&1
summ gpurun_out/r6c_c4.json "c4 auto"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_persistent -s 4 -c 1 \
   -o gpurun_out/prof_r6c_cfg3_k_pcg_persistent python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/ncu_r6c.log 2>&1
tail -3 gpurun_out/ncu_r6c.log
