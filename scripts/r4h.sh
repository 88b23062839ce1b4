set -x
mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'])
" $1 "$2"; }
timeout 1500 python -m pytest tests/test_gpu_gamg.py -q -rf -x > gpurun_out/r4h_gamg.log 2>&1
tail -3 gpurun_out/r4h_gamg.log
for tail in 0 4096 16384; do
LFOAM_LIB=liblfoam_gt.so LF_GAMG_TAIL=$tail timeout 300 python bench.py --steps 2 --warmup 3 --repeats 1 --precond GAMG --no-cpu-baseline > gpurun_out/r4h_gamg_timing_$tail.log 2>&1
grep LF_GAMG gpurun_out/r4h_gamg_timing_$tail.log | head -1
done
for cfg in 2 3; do
timeout 300 python bench.py --steps 10 --warmup 3 --repeats 2 --config $cfg --precond GAMG --no-cpu-baseline > gpurun_out/r4h_gamg_cfg$cfg.json 2>&1
summ gpurun_out/r4h_gamg_cfg$cfg.json "gamg cfg$cfg"
done
