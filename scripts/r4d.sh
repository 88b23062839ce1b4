# round-2 first GPU check of c5d876b: new tests, bench config 3, variant matrix, full suite
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_hbm.py tests/test_gpu_p2p.py tests/test_gpu_dic.py -q -rf > gpurun_out/r4d_new.log 2>&1
tail -15 gpurun_out/r4d_new.log
timeout 400 python bench.py --steps 20 --warmup 5 --repeats 3 --no-cpu-baseline > gpurun_out/r4d_cfg3.json 2> gpurun_out/r4d_cfg3.err
tail -c 1500 gpurun_out/r4d_cfg3.json; tail -5 gpurun_out/r4d_cfg3.err
for lib in liblfoam.so liblfoam_w0.so liblfoam_w0p0.so; do
  for lab in compressed int32; do
    LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline --labels $lab > gpurun_out/r4d_${lib}_${lab}.json 2>&1
    python -c "
import json
for l in open('gpurun_out/r4d_${lib}_${lab}.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$lib $lab', round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(d['roofline']['frac'],3), d['config']['pcg_iterations_per_step'])
"
  done
done
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/r4d_timing3.log 2>&1
grep -h "LF_TIMING" gpurun_out/r4d_timing3.log | head -8
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r4d_gpu.log 2>&1
tail -8 gpurun_out/r4d_gpu.log
