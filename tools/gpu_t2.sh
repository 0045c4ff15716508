for fr in 1e-12 1e-10 1e-8; do
echo "failrel $fr" >> gpurun_out/admm_fr.txt
PSDPROJ_CHOL_FAILREL=$fr timeout 300 python -m pytest tests/test_admm.py -m gpu -q 2>&1 | tail -2 >> gpurun_out/admm_fr.txt
PSDPROJ_CHOL_FAILREL=$fr PSDPROJ_TRI_NOREG=1 timeout 300 python -m pytest tests/test_admm.py -m gpu -q 2>&1 | tail -2 >> gpurun_out/admm_fr.txt
done
