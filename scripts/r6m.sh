mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hbm.py -q -x -k "runtime or prefetch or psi" > gpurun_out/r6m_tests.log 2>&1; tail -2 gpurun_out/r6m_tests.log
for rep in 1 2; do
for o in "dynamic_trips=0" "dynamic_trips=25" "dynamic_trips=40" "dynamic_trips=60"; do
  timeout 300 python scripts/step_trend.py 30 3 $o > gpurun_out/r6m_${o}_$rep.log 2>&1
  python -c "
l=[x for x in open('gpurun_out/r6m_${o}_$rep.log') if 'per step:' in x][0]; v=[float(x) for x in l.split('per step:')[1].split()]; print('$o', 'mean us/it %.1f' % (sum(v[5:])/len(v[5:])))"
done
done
