mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_m.log 2>&1; echo rc=$? >> gpurun_out/pytest_m.log
for w in cfg2 cfg3_c64 cfg3_c128; do timeout 300 python tools/kbench.py --workload $w --algos tc_pipe,tc_sp --only fused --iters 20 >> gpurun_out/kbench_m.log 2>&1; done
for e in 70 76 82 88 94; do echo "enc=$e" >> gpurun_out/kbench_m.log; ITLUMM_SP_ENC_CTAS=$e timeout 300 python tools/kbench.py --workload cfg2 --algos tc_sp --only fused --iters 20 >> gpurun_out/kbench_m.log 2>&1; done
