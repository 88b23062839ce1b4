mkdir -p gpurun_out
avg() { python -c "
l=[x for x in open('$1') if 'per step:' in x][0]; v=[float(x) for x in l.split('per step:')[1].split()]; print('$2', 'mean us/it %.1f' % (sum(v[3:])/len(v[3:])))"; }
for rep in 1 2; do
for lib in r5 nodyn cur; do
  L=liblfoam_$lib.so; [ $lib = cur ] && L=liblfoam.so
  LFOAM_LIB=$L timeout 600 python scripts/step_trend.py 12 N300 > gpurun_out/r6z.log 2>&1; avg gpurun_out/r6z.log "300 $lib"
  LFOAM_LIB=$L timeout 600 python scripts/step_trend.py 12 3 > gpurun_out/r6z.log 2>&1; avg gpurun_out/r6z.log "200 $lib"
done
done
for lib in r5 nodyn cur; do
  L=liblfoam_$lib.so; [ $lib = cur ] && L=liblfoam.so
  LFOAM_LIB=$L timeout 900 python scripts/step_trend.py 6 N400 > gpurun_out/r6z.log 2>&1; avg gpurun_out/r6z.log "400 $lib"
done
