# GAMG on the GPU (new), W88=2 variant, ncu source-level profile of the 200^3 solve
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gamg.py -q -rf > gpurun_out/r4e_gamg.log 2>&1
tail -30 gpurun_out/r4e_gamg.log
for cfg in 2 3; do
  timeout 600 python bench.py --steps 10 --warmup 3 --repeats 2 --config $cfg --precond GAMG --no-cpu-baseline > gpurun_out/r4e_gamg_cfg$cfg.json 2> gpurun_out/r4e_gamg_cfg$cfg.err
  tail -c 2500 gpurun_out/r4e_gamg_cfg$cfg.json; tail -3 gpurun_out/r4e_gamg_cfg$cfg.err
done
for lib in liblfoam.so liblfoam_w2.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r4e_${lib}.json 2>&1
  python -c "
import json
for l in open('gpurun_out/r4e_${lib}.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$lib', round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(d['roofline']['frac'],3), d['config']['pcg_iterations_per_step'])
"
done
LFOAM_LIB=liblfoam_w2.so timeout 600 python -m pytest tests/test_gpu_hbm.py -q -x -k "psi_every or compressed" > gpurun_out/r4e_w2_tests.log 2>&1; tail -3 gpurun_out/r4e_w2_tests.log
BENCH="python bench.py --steps 3 --warmup 3 --repeats 1 --config 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'k_(assemble|sum|pcg)' --csv --log-file gpurun_out/launches_r4e_cfg3.csv $BENCH > gpurun_out/ncu_launch_r4e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_persistent -s 2 -c 1 \
   -o gpurun_out/prof_r4e_cfg3_k_pcg_persistent $BENCH > gpurun_out/ncu_k_pcg_r4e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_gamg -s 2 -c 1 \
   -o gpurun_out/prof_r4e_cfg3_k_pcg_gamg $BENCH --precond GAMG > gpurun_out/ncu_k_gamg_r4e.log 2>&1
ls -la gpurun_out | tail
