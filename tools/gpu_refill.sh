# step time vs the ray-queue refill threshold (SPARROW_REFILL_MIN)
for rep in 1 2; do
  for r in 16 24 32 40 48; do
    v=$(SPARROW_REFILL_MIN=$r timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f %.4f' % (d['ms_per_step'], d['per_step_ms']['median']))")
    echo "refill_min=$r step(mean,median) $v" | tee -a gpurun_out/refill.txt
  done
done
