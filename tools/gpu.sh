#!/bin/bash
# One parameterised GPU-box script (replaces round 1's per-call run*.sh).  Run under gpurun:
#   gpurun --timeout S -- 'bash tools/gpu.sh TAG STEP [STEP ...]'
# Every log lands in gpurun_out/TAG_<step>.log.  Steps:
#   build          compile the libraries (they also travel in-tree)
#   tests          pytest -m gpu (whole GPU suite)
#   tests:EXPR     pytest -m gpu -k EXPR
#   file:PATH      pytest -m gpu PATH
#   smoke          __graft_entry__.smoke()
#   bench1         python bench.py (N = 1, defaults)
#   benchN:N       torchrun N ranks of bench.py --gpus N
#   ref            bench.py --impl reference
#   launches       ncu launch list (gpu__time_duration) of the N = 1 bench
#   ncu:REGEX      ncu --set full of the first launch of kernel REGEX in the N = 1 bench
#   py:SCRIPT,ARGS python SCRIPT (args after the colon, comma separated)
#   trun:N,SCRIPT,ARGS   torchrun N ranks of SCRIPT (comma separated)
#   env:K=V        export K=V for the following steps
#   sh:CMD         any shell command (commas become spaces)
TAG=$1; shift
mkdir -p gpurun_out
PORT=29700
for step in "$@"; do
  name=${step%%:*}; arg=${step#*:}; [ "$arg" = "$step" ] && arg=""
  log=gpurun_out/${TAG}_${name}${arg:+_$(echo "$arg" | tr -c 'A-Za-z0-9\n' '_')}.log
  echo "== $step -> $log"
  case $name in
    build)    timeout 600 python paper_2602_18007_b200/build.py > "$log" 2>&1 ;;
    tests)    if [ -n "$arg" ]; then timeout 2400 python -m pytest tests -m gpu -q -k "$arg" > "$log" 2>&1
              else timeout 2400 python -m pytest tests -m gpu -q --durations=25 > "$log" 2>&1; fi ;;
    file)     timeout 2400 python -m pytest "$arg" -m gpu -q --durations=15 > "$log" 2>&1 ;;
    smoke)    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$log" 2>&1 ;;
    bench1)   timeout 600 python bench.py > "$log" 2>&1 ;;
    benchN)   PORT=$((PORT+1)); timeout 600 python -m torch.distributed.run --nnodes=1 \
                --nproc-per-node "$arg" --master-addr 127.0.0.1 --master-port $PORT \
                bench.py --gpus "$arg" > "$log" 2>&1 ;;
    ref)      timeout 600 python bench.py --impl reference > "$log" 2>&1 ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
                --log-file gpurun_out/${TAG}_launches_n1.csv python bench.py --steps 2 --warmup 3 \
                --no-e2e --no-cpu-baseline --no-b1 --no-ring > "$log" 2>&1 ;;
    ncu)      timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$arg" \
                -s 4 -c 1 -o gpurun_out/${TAG}_prof_$(echo "$arg" | tr -c 'A-Za-z0-9\n' '_') \
                python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-b1 --no-ring > "$log" 2>&1 ;;
    py)       timeout 1200 python ${arg//,/ } > "$log" 2>&1 ;;
    trun)     PORT=$((PORT+1)); n=${arg%%,*}; rest=${arg#*,}
              timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" \
                --master-addr 127.0.0.1 --master-port $PORT ${rest//,/ } > "$log" 2>&1 ;;
    env)      export "$arg"; echo "export $arg" > "$log" ;;
    sh)       timeout 1200 bash -c "${arg//,/ }" > "$log" 2>&1 ;;
    *)        echo "unknown step $step" > "$log" ;;
  esac
  echo "rc=$?" >> "$log"
  tail -3 "$log"
done
true
