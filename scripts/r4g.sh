# cp.async pipeline variants of the diagonal solve; GAMG per-pass timing
set -x
mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'])
" $1 "$2"; }
for lib in liblfoam.so liblfoam_cpa.so liblfoam_cpaq.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r4g_${lib}.json 2>&1
  summ gpurun_out/r4g_${lib}.json $lib
done
LFOAM_LIB=liblfoam_cpa.so timeout 900 python -m pytest tests/test_gpu_hbm.py -q -x > gpurun_out/r4g_cpa_tests.log 2>&1; tail -2 gpurun_out/r4g_cpa_tests.log
LFOAM_LIB=liblfoam_gt.so timeout 300 python bench.py --steps 2 --warmup 3 --repeats 1 --precond GAMG --no-cpu-baseline > gpurun_out/r4g_gamg_timing.log 2>&1
grep LF_GAMG gpurun_out/r4g_gamg_timing.log | head -3
LFOAM_LIB=liblfoam_gt.so LF_GAMG_TAIL=0 timeout 300 python bench.py --steps 2 --warmup 3 --repeats 1 --precond GAMG --no-cpu-baseline > gpurun_out/r4g_gamg_timing_t0.log 2>&1
grep LF_GAMG gpurun_out/r4g_gamg_timing_t0.log | head -2
