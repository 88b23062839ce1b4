mkdir -p gpurun_out/protocol
timeout 1500 python scripts/protocol.py --meshes S,M --repeats 5 --out gpurun_out/protocol/protocol_r6_diag5.md > gpurun_out/protocol/protocol_r6_diag5.log 2>&1; tail -3 gpurun_out/protocol/protocol_r6_diag5.log
timeout 2400 python scripts/protocol.py --meshes L,XL --repeats 1 --out gpurun_out/protocol/protocol_r6_diag.md > gpurun_out/protocol/protocol_r6_diag.log 2>&1; tail -3 gpurun_out/protocol/protocol_r6_diag.log
