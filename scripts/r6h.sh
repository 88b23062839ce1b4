mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(sys.argv[2], round(d['ms_per_step'],2), [round(v/1e6,1) for v in d['repeats']['values']], round(r['frac'],3), d['config']['pcg_iterations_per_step']['mean'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" $1 "$2"; }
for lib in bulkT timing; do
LFOAM_LIB=liblfoam_$lib.so timeout 300 python bench.py --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline > gpurun_out/r6h_$lib.log 2>&1
grep -h "LF_TIMING block\|LF_BARRIER" gpurun_out/r6h_$lib.log | head -4
done
for rep in 1 2; do
for lib in bulk ""; do
  LFOAM_LIB=liblfoam${lib:+_$lib}.so timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/r6h_${lib}_$rep.json 2>&1
  summ gpurun_out/r6h_${lib}_$rep.json "c3 $lib"
done
done
