mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
for rep in 1 2; do
for lib in liblfoam_acq.so liblfoam.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r6d_${lib}_c3_$rep.json 2>&1
  summ gpurun_out/r6d_${lib}_c3_$rep.json "$lib c3"
done
done
for lib in liblfoam_acq.so liblfoam.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r6d_${lib}_c2.json 2>&1
  summ gpurun_out/r6d_${lib}_c2.json "$lib c2"
  LFOAM_LIB=$lib timeout 300 python bench.py --precond DIC --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline > gpurun_out/r6d_${lib}_c3dic.json 2>&1
  summ gpurun_out/r6d_${lib}_c3dic.json "$lib c3 DIC"
  LFOAM_LIB=$lib timeout 300 python bench.py --precond GAMG --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline > gpurun_out/r6d_${lib}_c3gamg.json 2>&1
  summ gpurun_out/r6d_${lib}_c3gamg.json "$lib c3 GAMG"
  LFOAM_LIB=$lib timeout 600 python bench.py --config 4 --steps 4 --warmup 3 --repeats 2 --no-cpu-baseline > gpurun_out/r6d_${lib}_c4.json 2>&1
  summ gpurun_out/r6d_${lib}_c4.json "$lib c4"
done
timeout 1200 python -m pytest tests/test_gpu_hbm.py tests/test_gpu_parity.py tests/test_gpu_dic.py tests/test_gpu_gamg.py tests/test_gpu_p2p.py -q -x > gpurun_out/r6d_tests.log 2>&1; tail -2 gpurun_out/r6d_tests.log
