mkdir -p gpurun_out
nvidia-smi -q | grep -i -A3 'gpc\|Bus Id' | head -5
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline > gpurun_out/r6f_c3.log 2>&1
grep -h "LF_TIMING block\|LF_BARRIER" gpurun_out/r6f_c3.log | head -4
python - <<'PY'
import re
for l in open('gpurun_out/r6f_c3.log'):
    if l.startswith('LF_ARRIVALS'):
        head, vals = l.split(':', 1)
        v = [float(x) for x in vals.split()]
        G = len(v)
        print(head, 'G', G, 'mean %.1f' % (sum(v)/G), 'max %.1f' % max(v))
        # by block id mod 148 pairs and sorted slow list
        slow = sorted(range(G), key=lambda b: -v[b])[:30]
        print(' slowest', [(b, v[b]) for b in slow])
        hist = [0]*12
        for x in v: hist[min(int(x//5), 11)] += 1
        print(' hist(5us bins)', hist)
PY
