# variant matrix at config 3: w88 x psi2 x labels
for lib in liblfoam.so liblfoam_w0.so liblfoam_w0p0.so; do
  for lab in compressed int32; do
    echo "== $lib $lab"
    LFOAM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline --labels $lab > gpurun_out/r4c_${lib}_${lab}.json 2>&1
    python -c "
import json,sys
for l in open('gpurun_out/r4c_${lib}_${lab}.json'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],2), d['repeats']['values'], d['roofline']['frac'])
"
  done
done
