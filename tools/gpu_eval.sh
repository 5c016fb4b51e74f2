mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_evaluate.py tests/test_gpu_asl.py -x -q > gpurun_out/t_eval.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_eval.log
timeout 300 python tools/bench_learner.py > gpurun_out/learner.jsonl 2> gpurun_out/learner.err
timeout 600 python tools/bench_eval.py > gpurun_out/eval.jsonl 2> gpurun_out/eval.err
timeout 200 python tools/bench_asl.py --seconds 20 > gpurun_out/asl_graph.json 2> gpurun_out/asl_graph.err
