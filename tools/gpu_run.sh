#!/bin/bash
# One gpurun command for the common measurement steps (run from the repo root on
# the GPU box):  tools/gpu_run.sh STEP [STEP ...]
#   tests[:EXPR]   pytest -m gpu (optionally -k EXPR)      -> gpurun_out/tests.log
#   smoke          __graft_entry__.smoke()                  -> gpurun_out/smoke.log
#   bench[:ARGS]   python bench.py ARGS (default N=1)       -> gpurun_out/bench*.json
#   ref            bench.py --impl reference                -> gpurun_out/bench_ref.json
#   launches       ncu launch list of the default bench    -> gpurun_out/launches.csv
#   py:SCRIPT ARGS python SCRIPT ARGS                       -> gpurun_out/<script>.json
#   dbench:N:ARGS  torchrun of bench.py on N GPUs           -> gpurun_out/dbench_N_*.json
# Exit codes of every step go to gpurun_out/rc.txt.
mkdir -p gpurun_out
python -c "from paper_2510_19262_b200 import build as b; b.build()" > gpurun_out/build.log 2>&1
for step in "$@"; do
  name="${step%%:*}"; arg="${step#*:}"; [ "$arg" = "$step" ] && arg=""
  case "$name" in
    tests)
      if [ -n "$arg" ]; then k=(-k "$arg"); else k=(); fi
      timeout 2400 python -m pytest tests -m gpu -q -rfs --timeout 900 "${k[@]}" > gpurun_out/tests.log 2>&1 ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 ;;
    bench)
      tag=$(echo "$arg" | tr -c 'a-zA-Z0-9\n' '_')
      timeout 1200 python bench.py $arg > "gpurun_out/bench${tag:+_$tag}.json" 2> "gpurun_out/bench${tag:+_$tag}.err" ;;
    ref)
      timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err ;;
    launches)
      timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-graph $arg \
        > gpurun_out/launches.log 2>&1 ;;
    dbench)
      n="${arg%%:*}"; rest="${arg#*:}"; [ "$rest" = "$arg" ] && rest=""
      tag=$(echo "$rest" | tr -c 'a-zA-Z0-9\n' '_')
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus "$n" $rest \
        > "gpurun_out/dbench_${n}${tag:+_$tag}.json" 2> "gpurun_out/dbench_${n}${tag:+_$tag}.err" ;;
    py)
      scr="${arg%% *}"; rest="${arg#* }"; [ "$rest" = "$arg" ] && rest=""
      out=$(basename "$scr" .py)
      timeout 1500 python $scr $rest > "gpurun_out/$out.json" 2> "gpurun_out/$out.err" ;;
    *) echo "unknown step $step" ;;
  esac
  echo "$step rc=$?" >> gpurun_out/rc.txt
done
echo finished >> gpurun_out/rc.txt
