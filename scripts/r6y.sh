mkdir -p gpurun_out
avg() { python -c "
l=[x for x in open('$1') if 'per step:' in x][0]; v=[float(x) for x in l.split('per step:')[1].split()]; print('$2', 'mean us/it %.1f' % (sum(v[3:])/len(v[3:])))"; }
for rep in 1 2; do
LFOAM_LIB=liblfoam_r5.so timeout 600 python scripts/step_trend.py 12 N300 > gpurun_out/r6y_r5_300.log 2>&1; avg gpurun_out/r6y_r5_300.log "300 r5build"
timeout 600 python scripts/step_trend.py 12 N300 > gpurun_out/r6y_cur_300.log 2>&1; avg gpurun_out/r6y_cur_300.log "300 current"
timeout 600 python scripts/step_trend.py 12 N300 l2_prefetch=2 > gpurun_out/r6y_nopf_300.log 2>&1; avg gpurun_out/r6y_nopf_300.log "300 current pf-off"
timeout 600 python scripts/step_trend.py 12 N300 l2_prefetch=2 dynamic_trips=0 > gpurun_out/r6y_none_300.log 2>&1; avg gpurun_out/r6y_none_300.log "300 current pf-off dyn0"
done
LFOAM_LIB=liblfoam_r5.so timeout 900 python scripts/step_trend.py 6 N400 > gpurun_out/r6y_r5_400.log 2>&1; avg gpurun_out/r6y_r5_400.log "400 r5build"
timeout 900 python scripts/step_trend.py 6 N400 > gpurun_out/r6y_cur_400.log 2>&1; avg gpurun_out/r6y_cur_400.log "400 current"
timeout 900 python scripts/step_trend.py 6 N400 dynamic_trips=0 > gpurun_out/r6y_d0_400.log 2>&1; avg gpurun_out/r6y_d0_400.log "400 current dyn0"
