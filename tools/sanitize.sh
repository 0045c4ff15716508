# compute-sanitizer evidence for the hand-rolled synchronisation (mbarrier / DSMEM / st.async in the
# cluster tridiagonalisation and Cholesky, the tile kernel's barriers, the residency flag).
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck; do
  for args in "eigh 60 20" "eigh 200 60" "eigh 400 120" "chol 300" "c1"; do
    tag=$(echo $args | tr ' ' '_')
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_case.py $args > $OUT/${tool}_$tag.log 2>&1
    echo "$tool $args rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $OUT/${tool}_$tag.log | tail -2 | tr '\n' ' ')"
  done
done > $OUT/summary.txt
timeout 900 $CS --tool memcheck --print-limit 20 python tools/sanitize_case.py c1 > $OUT/memcheck_c1.log 2>&1
echo "memcheck c1 rc=$? $(grep 'ERROR SUMMARY' $OUT/memcheck_c1.log)" >> $OUT/summary.txt
cat $OUT/summary.txt
