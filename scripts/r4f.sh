# GAMG V-cycle with stored x/z (one gather per neighbour), q-recurrence variants, tail sweep
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gamg.py -q -rf -x > gpurun_out/r4f_gamg.log 2>&1
tail -5 gpurun_out/r4f_gamg.log
LFOAM_LIB=liblfoam_qrec.so timeout 1500 python -m pytest tests/test_gpu_hbm.py tests/test_gpu_fullsize.py -q -rf -x > gpurun_out/r4f_qrec_tests.log 2>&1
tail -5 gpurun_out/r4f_qrec_tests.log
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'])
" $1 "$2"; }
for lib in liblfoam.so liblfoam_qrec.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r4f_${lib}.json 2>&1
  summ gpurun_out/r4f_${lib}.json $lib
done
for tail in 0 2048 4096 16384 65536; do
  LF_GAMG_TAIL=$tail timeout 300 python bench.py --steps 5 --warmup 3 --repeats 2 --precond GAMG --no-cpu-baseline > gpurun_out/r4f_gamg_t$tail.json 2>&1
  summ gpurun_out/r4f_gamg_t$tail.json "gamg tail $tail"
done
LFOAM_LIB=liblfoam_gq0.so timeout 300 python bench.py --steps 5 --warmup 3 --repeats 2 --precond GAMG --no-cpu-baseline > gpurun_out/r4f_gamg_gq0.json 2>&1
summ gpurun_out/r4f_gamg_gq0.json "gamg qrec0"
timeout 300 python bench.py --steps 10 --warmup 3 --repeats 2 --config 2 --precond GAMG --no-cpu-baseline > gpurun_out/r4f_gamg_cfg2.json 2>&1
summ gpurun_out/r4f_gamg_cfg2.json "gamg cfg2"
BENCH="python bench.py --steps 3 --warmup 3 --repeats 1 --config 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_gamg -s 2 -c 1 \
   -o gpurun_out/prof_r4f_cfg3_k_pcg_gamg $BENCH --precond GAMG > gpurun_out/ncu_k_gamg_r4f.log 2>&1
