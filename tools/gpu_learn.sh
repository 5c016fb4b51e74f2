mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_asl.py -q > gpurun_out/t_learn.log 2>&1; echo "rc=$?" >> gpurun_out/t_learn.log
timeout 300 python tools/bench_learner.py > gpurun_out/learner2.jsonl 2> gpurun_out/learner2.err
timeout 200 python tools/bench_asl.py --seconds 20 > gpurun_out/asl_fused.json 2> gpurun_out/asl_fused.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"ddqn_" -s 40 -c 2 -o gpurun_out/prof_learn python tools/bench_learner.py --updates 50 --reference-updates 1 > gpurun_out/ncu_learn.log 2>&1
