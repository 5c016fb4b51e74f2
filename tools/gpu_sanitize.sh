# compute-sanitizer pass over the step kernel (4,096 and 65,536 envs, plus a
# reset-heavy timeout config) and the replay kernels: racecheck, synccheck,
# memcheck, initcheck.  Logs -> gpurun_out/sanitize_<tool>.log
tag=${1:-r02}
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 99 \
    python tools/debug/sanitize_workload.py > gpurun_out/sanitize_${tool}_$tag.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary_$tag.txt
done
cat gpurun_out/sanitize_summary_$tag.txt
