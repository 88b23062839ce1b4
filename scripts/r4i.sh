set -x
mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
for rep in 1 2; do
for lib in liblfoam.so liblfoam_pf1.so liblfoam_pf2.so liblfoam_u4.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r4i_${lib}_$rep.json 2>&1
  summ gpurun_out/r4i_${lib}_$rep.json $lib
done
done
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/r4i_timing3.log 2>&1
grep -h "LF_TIMING" gpurun_out/r4i_timing3.log | head -4
LFOAM_LIB=liblfoam_pf2.so timeout 900 python -m pytest tests/test_gpu_hbm.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r4i_pf2_tests.log 2>&1; tail -2 gpurun_out/r4i_pf2_tests.log
