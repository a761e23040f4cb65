# ncu evidence of one round (run on the GPU box from the repo root):
#   bash tools/tuning/prof2.sh r02
# one `ncu --set full` capture per native leaf at its bench size, then the
# launch list (durations only) of the bench command; summarise here with
#   python tools/tuning/ncu_summary.py r02 ; python tools/tuning/launch_shares.py r02
R=${1:-r02}
set -x
mkdir -p gpurun_out
for k in gemm ttv innerprod ttm mttkrp g1; do python tools/tuning/prof2.py $k || exit 1; done
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s 1 -c 1 -o gpurun_out/${R}_dgemm python tools/tuning/prof2.py gemm > gpurun_out/ncu_${R}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ttv_bulk -s 1 -c 1 -o gpurun_out/${R}_ttv python tools/tuning/prof2.py ttv >> gpurun_out/ncu_${R}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:innerprod_bulk -s 1 -c 1 -o gpurun_out/${R}_innerprod python tools/tuning/prof2.py innerprod >> gpurun_out/ncu_${R}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s 1 -c 1 -o gpurun_out/${R}_ttm python tools/tuning/prof2.py ttm >> gpurun_out/ncu_${R}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mttkrp_st_kernel -s 1 -c 1 -o gpurun_out/${R}_mttkrp python tools/tuning/prof2.py mttkrp >> gpurun_out/ncu_${R}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_grouped -s 4 -c 1 -o gpurun_out/${R}_g1 python tools/tuning/prof2.py g1 >> gpurun_out/ncu_${R}.log 2>&1
python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_plain_${R}.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_bench_${R}.log 2>&1
echo done
