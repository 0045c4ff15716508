mkdir -p gpurun_out
python tools/gemm_probe.py > gpurun_out/gemm.log 2>&1
PSDPROJ_GEMM_TILE=128 python tools/gemm_probe.py >> gpurun_out/gemm.log 2>&1
