mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_y.log 2>&1; echo rc=$? >> gpurun_out/pytest_y.log
timeout 300 python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san_memcheck.log 2>&1
echo rc=$? >> gpurun_out/san_memcheck.log
