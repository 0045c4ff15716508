mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/tridbg.txt
for d in 0 64; do
  echo "dbg=$d" >> gpurun_out/tridbg.txt
  PSDPROJ_TRI_DBG=$d PSDPROJ_TRI_PROF=1 timeout 60 python tools/eigh_probe.py 200:70,400:130 2>&1 | grep "rank\|ms\|owner" >> gpurun_out/tridbg.txt
done
