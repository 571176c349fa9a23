# compute-sanitizer gate (SURVEY §5 race detection): memcheck, racecheck and synccheck over the
# tools/sanitize_driver.py workloads on ONE GPU. Logs: gpurun_out/sanitize_<tool>_<mode>.log;
# summary: gpurun_out/sanitize_summary.txt (copy to profiles/ to commit).
mkdir -p gpurun_out
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  for mode in ${MODES:-walled periodic fp32 slab shard_local}; do
    log=gpurun_out/sanitize_${tool}_${mode}.log
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
        python tools/sanitize_driver.py $mode > $log 2>&1
    rc=$?
    summ=$(grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|LEAK SUMMARY" $log | sort | uniq -c | tr '\n' ';')
    ok=$(grep -c "sanitize_driver $mode: ok" $log)
    echo "$tool $mode rc=$rc driver_ok=$ok $summ" | tee -a gpurun_out/sanitize_summary.txt
  done
done
