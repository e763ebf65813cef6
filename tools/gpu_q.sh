mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_q.log 2>&1; echo rc=$? >> gpurun_out/pytest_q.log
timeout 600 python bench.py > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo rc=$? >> gpurun_out/bench_q.err
