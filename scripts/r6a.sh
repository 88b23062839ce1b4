set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
for rep in 1 2; do
for lib in liblfoam_base.so liblfoam_lpf1.so liblfoam_lpf2.so liblfoam_lpf1b.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline > gpurun_out/r6a_${lib}_$rep.json 2>&1
  summ gpurun_out/r6a_${lib}_$rep.json $lib
done
done
LFOAM_LIB=liblfoam_lpf1b.so timeout 900 python -m pytest tests/test_gpu_hbm.py -q -x > gpurun_out/r6a_tests.log 2>&1; tail -2 gpurun_out/r6a_tests.log
