#!/bin/bash
# Round-closing ncu evidence (one GPU): the launch list of the C3 bench step and
# full captures of the top kernels.  Every profiled command first ran without ncu.
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-graph --no-extra"
$B > gpurun_out/plain_bench.json 2> gpurun_out/plain_bench.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/rc.txt
python tools/sched_bench.py --only c3 > gpurun_out/sb3.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_hist_rank" -s 6 -c 1 \
      -o gpurun_out/ncu_c3_hist python tools/sched_bench.py --only c3 > gpurun_out/ncu_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_node" -s 6 -c 1 \
      -o gpurun_out/ncu_c3_node python tools/sched_bench.py --only c3 >> gpurun_out/ncu_c3.log 2>&1
echo "c3 rc=$?" >> gpurun_out/rc.txt
python tools/sched_bench.py --only c4 > gpurun_out/sb4.json 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"k_chunk_sort|k_lpt_wstage|k_expand|k_eval_node" -s 12 -c 4 \
      -o gpurun_out/ncu_c4_sched python tools/sched_bench.py --only c4 > gpurun_out/ncu_c4.log 2>&1
echo "c4 rc=$?" >> gpurun_out/rc.txt
ncu --set full --clock-control none -k regex:k_pack -s 3 -c 1 -o gpurun_out/ncu_pack $B \
    > gpurun_out/ncu_pack.log 2>&1
echo "pack rc=$?" >> gpurun_out/rc.txt
echo finished >> gpurun_out/rc.txt
