mkdir -p gpurun_out
avg() { python -c "
l=[x for x in open('$1') if 'per step:' in x][0]; v=[float(x) for x in l.split('per step:')[1].split()]; print('$2', 'mean us/it %.1f' % (sum(v[3:])/len(v[3:])))"; }
for rep in 1 2; do
for lib in r5 nodyn nodyn_acq nodyn_nolpf nodyn_nolpf_acq; do
  LFOAM_LIB=liblfoam_$lib.so timeout 600 python scripts/step_trend.py 10 N300 > gpurun_out/r6za.log 2>&1; avg gpurun_out/r6za.log "300 $lib"
done
done
for lib in r5 nodyn nodyn_acq nodyn_nolpf nodyn_nolpf_acq; do
  LFOAM_LIB=liblfoam_$lib.so timeout 900 python scripts/step_trend.py 6 N400 > gpurun_out/r6za.log 2>&1; avg gpurun_out/r6za.log "400 $lib"
done
