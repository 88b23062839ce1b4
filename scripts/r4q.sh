set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gamg.py -q -rf -x > gpurun_out/r4q_gamg.log 2>&1
tail -3 gpurun_out/r4q_gamg.log
for tail in 0 4096; do
LFOAM_LIB=liblfoam_gt.so LF_GAMG_TAIL=$tail timeout 300 python bench.py --steps 2 --warmup 3 --repeats 1 --precond GAMG --no-cpu-baseline > gpurun_out/r4q_gamg_timing_$tail.log 2>&1
grep LF_GAMG gpurun_out/r4q_gamg_timing_$tail.log | head -1
done
timeout 300 python bench.py --steps 10 --warmup 3 --repeats 2 --precond GAMG --no-cpu-baseline > gpurun_out/r4q_gamg_cfg3.json 2>&1
python -c "
import json
for l in open('gpurun_out/r4q_gamg_cfg3.json'):
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], d['roofline']['frac'], d['config']['pcg_iterations_per_step'])"
