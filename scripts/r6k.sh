mkdir -p gpurun_out
for o in "dynamic_trips=0" "dynamic_trips=40" "dynamic_trips=70"; do
  for lib in ut4 ut8; do
  LFOAM_LIB=liblfoam_$lib.so timeout 300 python scripts/step_trend.py 30 3 $o > gpurun_out/r6k_${lib}_$o.log 2>&1
  python -c "
l=[x for x in open('gpurun_out/r6k_${lib}_$o.log') if 'per step:' in x][0]; v=[float(x) for x in l.split('per step:')[1].split()]; print('$lib', '$o', 'mean us/it %.1f' % (sum(v[5:])/len(v[5:])))"
  done
done
