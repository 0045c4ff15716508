mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
PSDPROJ_TRI_NOREG=1 timeout 300 python -m pytest tests/test_admm.py -m gpu -q > gpurun_out/gputests_noreg.log 2>&1; echo tests=$? >> gpurun_out/gputests_noreg.log
