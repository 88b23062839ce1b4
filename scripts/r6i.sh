mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
timeout 900 python -m pytest tests/test_gpu_hbm.py -q -x -k "dynamic or compressed or psi" > gpurun_out/r6i_tests.log 2>&1; tail -2 gpurun_out/r6i_tests.log
for d in 40 100; do
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline --dyn-pct $d > gpurun_out/r6i_t$d.log 2>&1
grep -h "LF_TIMING block\|LF_BARRIER" gpurun_out/r6i_t$d.log | head -4
done
for rep in 1 2; do
for d in 0 25 40 60 100; do
  timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline --dyn-pct $d > gpurun_out/r6i_d${d}_$rep.json 2>&1
  summ gpurun_out/r6i_d${d}_$rep.json "c3 dyn$d"
done
done
