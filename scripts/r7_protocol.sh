mkdir -p gpurun_out/protocol
timeout 900 python scripts/protocol.py --meshes S,M --repeats 5 --out gpurun_out/protocol/protocol_r7_diag5.md > gpurun_out/protocol/protocol_r7_diag5.log 2>&1; tail -2 gpurun_out/protocol/protocol_r7_diag5.log
timeout 1500 python scripts/protocol.py --meshes L,XL --repeats 1 --out gpurun_out/protocol/protocol_r7_diag.md > gpurun_out/protocol/protocol_r7_diag.log 2>&1; tail -2 gpurun_out/protocol/protocol_r7_diag.log
