mkdir -p gpurun_out
for o in "" "l2_prefetch=2" "dynamic_trips=40" "" "l2_prefetch=2"; do
  timeout 300 python scripts/step_trend.py 60 3 $o 2>&1 | tail -2
done
