#!/usr/bin/env bash
# Commands behind every round-2 file in profiles/ (run from the repo root on a
# B200 box; the multi-GPU ones need that many GPUs).  Each line writes to
# gpurun_out/; the committed profiles/ files are copies of those outputs.
set -euo pipefail
mkdir -p gpurun_out
N=${1:-1}

if [ "$N" = 1 ]; then
  python -m pytest tests -m gpu -q                                     # parity (1 GPU)
  python -c "import __graft_entry__ as g; g.smoke()"
  python bench.py --steps 5 --warmup 3          > gpurun_out/r02_bench_n1.log      # profiles/bench_r02_n1.jsonl
  python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_ref_n1.log # profiles/bench_r02_reference_n1.jsonl
  python tools/launch_latency.py                > gpurun_out/r02_latency.log      # profiles/launch_latency_r02.jsonl
  python tools/kernel_probe.py                                          # MTTKRP tail / TTM bare-call numbers
  python tools/mttkrp_clocks.py 18 19 22; MK_I=4096 python tools/mttkrp_clocks.py 18 19   # MTTKRP table (mttkrp.cu)
  python tools/mttkrp_configs.py 18 19 22                               # same bits across MTTKRP configurations
  TD_TTV_BULK=0 python tools/tuning/kperf.py ttv innerprod; python tools/tuning/kperf.py ttv innerprod  # load vs copy-engine staging
  bash tools/tuning/prof2.sh r02                                        # ncu captures + launch list
  python tools/tuning/ncu_summary.py r02                                # -> profiles/ncu_summary_r02.json
  python tools/tuning/launch_shares.py gpurun_out/r02_launches.csv profiles/launches_r02_bench_n1.json
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size \
      --clock-control none -k regex:Kernel2 -s 1 -c 1 python tools/cublas_traffic.py   # cublas_dgemm_traffic_r02.txt
else
  torchrun --nproc-per-node "$N" --master-addr 127.0.0.1 --master-port 29600 tests/mp_check.py
  torchrun --nproc-per-node "$N" --master-addr 127.0.0.1 --master-port 29601 tests/ref_suite_spmd.py
  torchrun --nproc-per-node "$N" --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus "$N" --steps 5 --warmup 3
  if [ "$N" = 4 ]; then
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus 4 --procs 8
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29604 bench.py --gpus 4 --procs 8 \
        --placement cyclic
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29606 bench.py --gpus 2   # bench_r02_n2.jsonl
    # copy-engine shifts off (NCCL send/recv): the comparison in DESIGN §1 item 3
    TD_CE_SHIFTS=0 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29607 bench.py --gpus 4 \
        --workload gemm --e2e-steps 1 --no-cpu-baseline
  fi
  if [ "$N" = 2 ]; then
    timeout 180 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29605 tests/nccl_watchdog_check.py
  fi
fi
