mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_t.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_t.csv $CMD > gpurun_out/ncu_t1.log 2>&1
echo rc=$? >> gpurun_out/ncu_t1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc|k_encode_rows' -s 6 -c 2 -o gpurun_out/prof_t $CMD > gpurun_out/ncu_t2.log 2>&1
echo rc=$? >> gpurun_out/ncu_t2.log
