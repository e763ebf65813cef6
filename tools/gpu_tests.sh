#!/bin/bash
# Full GPU suite + smoke (what the driver runs at round end), logs under gpurun_out/tests/.
mkdir -p gpurun_out/tests
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tests/smoke.log 2>&1; echo rc=$? >> gpurun_out/tests/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rs > gpurun_out/tests/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/tests/pytest_gpu.log
