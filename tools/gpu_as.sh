mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 > gpurun_out/pytest_as.log 2>&1; echo rc=$? >> gpurun_out/pytest_as.log
