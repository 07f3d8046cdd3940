#!/bin/bash
# Round-2 evidence: bench (K=20 burst + sustained + e2e), launch list and ncu --set full of the
# headline step, batched strategies, small-n latency, solver timings, C5 scale, sanitizer on smoke.
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-secondary --sustained-ms 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/launches_$TAG.csv gpurun_out/launches_$TAG > /dev/null 2>&1
bash scripts/gpu_ncu_one.sh pass1_$TAG k_pass1 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-secondary --sustained-ms 0 > /dev/null 2>&1
bash scripts/gpu_ncu_one.sh pass1norm_$TAG k_pass1 python scripts/p1_time.py --norm --reps 2 > /dev/null 2>&1
bash scripts/gpu_ncu_one.sh batched_$TAG k_batched python scripts/batched_time.py > /dev/null 2>&1
timeout 300 python scripts/batched_strategy_time.py > gpurun_out/batched_strat_$TAG.jsonl 2>&1
timeout 300 python scripts/latency.py > gpurun_out/latency_$TAG.jsonl 2>&1
( for n in 1000 10000 16384 32768 100000 1000000; do timeout 120 python scripts/step_graph_time.py $n; PIPE=four timeout 120 python scripts/step_graph_time.py $n; done ) > gpurun_out/step_graph_$TAG.jsonl 2>&1
( for n in 1000 10000 16384; do timeout 120 python scripts/small_phases.py $n; done ) > gpurun_out/small_phases_$TAG.jsonl 2>&1
timeout 300 python scripts/acg_breakdown.py > gpurun_out/acg_breakdown_$TAG.jsonl 2>&1
( for m in 0 32; do timeout 120 python scripts/p1_time.py --norm --mode $m; done; QDOT_B200_P1_NARROW=0 timeout 120 python scripts/p1_time.py --norm; timeout 120 python scripts/p1_time.py --norm --data illcond --eps 1e-12; timeout 120 python scripts/p1_time.py ) > gpurun_out/p1_norm_$TAG.jsonl 2>&1
timeout 300 python scripts/solver_bench.py > gpurun_out/solver_bench_$TAG.jsonl 2>&1
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke_$TAG.log 2>&1
timeout 600 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck_smoke_$TAG.log 2>&1
timeout 600 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/synccheck_smoke_$TAG.log 2>&1
cut -c1-300 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/memcheck_smoke_$TAG.log gpurun_out/racecheck_smoke_$TAG.log
echo done
