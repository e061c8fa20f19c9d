mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mc_build.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_paths.py > gpurun_out/r2_sanitizer_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitizer_memcheck.log
timeout 900 python -m pytest -q -m gpu tests/test_gpuarray_gpu.py tests/test_host_streaming_gpu.py tests/test_runtime_abi.py tests/test_reduction_gpu.py -p no:cacheprovider > gpurun_out/mc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mc_pytest.log
tail -n 3 gpurun_out/r2_sanitizer_memcheck.log gpurun_out/mc_pytest.log
