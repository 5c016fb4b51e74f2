# SP_CHECKED build (device-side bounds checks; compute-sanitizer is closed on
# this pool): the sanitize workload and the BASELINE-size parity tests.
tag=${1:-r02}
SPARROW_LIB_PATH=variants/checked.so timeout 900 python tools/debug/sanitize_workload.py > gpurun_out/checked_workload_$tag.log 2>&1
echo "workload rc=$?" >> gpurun_out/checked_$tag.txt
SPARROW_LIB_PATH=variants/checked.so timeout 1500 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_env.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/checked_tests_$tag.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/checked_tests_$tag.log)" >> gpurun_out/checked_$tag.txt
cat gpurun_out/checked_$tag.txt
