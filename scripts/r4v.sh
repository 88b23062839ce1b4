set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r4v_gpu.log 2>&1
tail -5 gpurun_out/r4v_gpu.log
BENCH="python bench.py --steps 3 --warmup 3 --repeats 1 --config 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'k_(assemble|sum|pcg)' --csv --log-file gpurun_out/launches_r4v_cfg3.csv $BENCH > gpurun_out/ncu_launch_r4v.log 2>&1
grep -i assemble gpurun_out/launches_r4v_cfg3.csv | head -6
