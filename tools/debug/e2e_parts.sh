# e2e of sp_env_step_host by row-part split (debug A/B; bench.py e2e leg only)
for rep in 1 2; do
for cfg in "4:" "3:1,2,5" "3:1,2,4" "3:3,5,8" "4:1,2,4,8" "2:1,3"; do
  P=${cfg%%:*}; W=${cfg#*:}
  if [ -n "$W" ]; then export SPARROW_HOST_PART_W=$W; else unset SPARROW_HOST_PART_W; fi
  SPARROW_HOST_PARTS=$P timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 40 --no-cpu-baseline --no-lidar --no-replay > gpurun_out/e2ep.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/e2ep.json').read().strip().splitlines()[-1]); e=j['e2e']; print('$cfg', round(e['value']/1e6,1), 'M', round(e['ms_per_step_mean'],4), round(e['per_step_ms']['median'],4))"
done; done
for cfg in "3:1,2,5" "3:3,5,8"; do
  P=${cfg%%:*}; W=${cfg#*:}
  SPARROW_HOST_PART_W=$W SPARROW_HOST_PARTS=$P SPARROW_LIB_PATH=variants/ht.so timeout 200 python tools/debug/host_timeline.py 2>&1 | tail -2
done
