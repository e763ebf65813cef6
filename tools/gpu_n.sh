mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_n.log 2>&1; echo rc=$? >> gpurun_out/pytest_n.log
for w in cfg2 cfg3_c64 cfg3_c128; do timeout 300 python tools/kbench.py --workload $w --algos tc_pipe,tc_sp --only fused --iters 20 >> gpurun_out/kbench_n.log 2>&1; done
for e in 64 72 80 88 96; do echo "enc=$e" >> gpurun_out/kbench_n.log; ITLUMM_SP_ENC_CTAS=$e timeout 300 python tools/kbench.py --workload cfg2 --algos tc_sp --only fused --iters 20 >> gpurun_out/kbench_n.log 2>&1; done
