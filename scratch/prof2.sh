set -x
for k in gemm ttv innerprod ttm mttkrp; do python scratch/prof2.py $k || exit 1; done
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s 1 -c 1 -o gpurun_out/r01_dgemm python scratch/prof2.py gemm > gpurun_out/ncu_r01.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ttv_kernel -s 1 -c 1 -o gpurun_out/r01_ttv python scratch/prof2.py ttv >> gpurun_out/ncu_r01.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:innerprod_partial -s 1 -c 1 -o gpurun_out/r01_innerprod python scratch/prof2.py innerprod >> gpurun_out/ncu_r01.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s 1 -c 1 -o gpurun_out/r01_ttm python scratch/prof2.py ttm >> gpurun_out/ncu_r01.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s 1 -c 1 -o gpurun_out/r01_mttkrp python scratch/prof2.py mttkrp >> gpurun_out/ncu_r01.log 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo done
