set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r4l_gpu.log 2>&1
tail -8 gpurun_out/r4l_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4l_smoke.log 2>&1; tail -3 gpurun_out/r4l_smoke.log
timeout 600 python bench.py > gpurun_out/r4l_bench.json 2> gpurun_out/r4l_bench.err; tail -c 600 gpurun_out/r4l_bench.json; tail -3 gpurun_out/r4l_bench.err
timeout 600 python scripts/p2p_overhead.py 200 5 > gpurun_out/r4l_p2p_overhead.json 2>&1; tail -3 gpurun_out/r4l_p2p_overhead.json
timeout 600 python scripts/p2p_overhead.py 100 10 > gpurun_out/r4l_p2p_overhead100.json 2>&1; tail -3 gpurun_out/r4l_p2p_overhead100.json
