timeout 900 python -m pytest tests/test_apps_gpu.py tests/test_reference_suite_gpu.py -x -q > gpurun_out/apps.log 2>&1; echo "rc=$?"
tail -30 gpurun_out/apps.log
timeout 600 ./build/ref_tests_on_b200 2>&1 | tail -4
