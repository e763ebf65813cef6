mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "mlp" > gpurun_out/pytest_u.log 2>&1; echo rc=$? >> gpurun_out/pytest_u.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_u2.log 2>&1; echo rc=$? >> gpurun_out/pytest_u2.log
