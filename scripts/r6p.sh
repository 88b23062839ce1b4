mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r6p_gpu_tests.log 2>&1; tail -3 gpurun_out/r6p_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6p_smoke.log 2>&1; tail -2 gpurun_out/r6p_smoke.log
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
for rep in 1 2; do
for lib in liblfoam.so liblfoam_spin0.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r6p_${lib}_$rep.json 2>&1
  summ gpurun_out/r6p_${lib}_$rep.json "c3 $lib"
done
done
