mkdir -p gpurun_out/ab
for v in "3 4" "4 0" "3 0" "4 1"; do set -- $v; echo "ST=$1 CS=$2" >> gpurun_out/ab/kb.txt; ITLUMM_TC_STAGES=$1 ITLUMM_TC_CS=$2 ITLUMM_PAIR=0 timeout 300 python tools/kbench.py --workload cfg5 --algos tc --only acc --iters 10 >> gpurun_out/ab/kb.txt 2>&1; done
