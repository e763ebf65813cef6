mkdir -p gpurun_out
timeout 300 python tools/kbench.py --workload cfg2 --algos simt > gpurun_out/kbench_cfg2.log 2>&1
timeout 300 python tools/kbench.py --workload cfg1 --algos simt >> gpurun_out/kbench_cfg2.log 2>&1
timeout 300 python tools/kbench.py --workload cfg3_c64 --algos simt >> gpurun_out/kbench_cfg2.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --algo simt --no-cpu-baseline --e2e-steps 3 > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lut -s 3 -c 1 -o gpurun_out/prof_simt_cfg2 python bench.py --steps 5 --warmup 3 --algo simt --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu3.log 2>&1
echo rc=$? >> gpurun_out/ncu3.log
