mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'], r['traffic'])
" $1 "$2"; }
for rep in 1 2; do
for lib in liblfoam.so liblfoam_pfl1.so; do
  LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r6t_${lib}_$rep.json 2>&1
  summ gpurun_out/r6t_${lib}_$rep.json "c3 $lib"
done
done
