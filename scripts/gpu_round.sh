#!/bin/bash
# Round evidence: smoke, all GPU tests (incl. slow), bench (+ reference arm), launch list,
# ncu --set full captures of k_pass1 (C2), k_batched (C4), k_pass1 (C3), k_exact (C2).
TAG=${1:-r1b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1400 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --steps 500 --warmup 10 --e2e-steps 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 \
   -o gpurun_out/pass1_$TAG python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-secondary > gpurun_out/ncu_pass1_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 3 -c 1 \
   -o gpurun_out/batched_$TAG python scripts/batched_time.py > gpurun_out/ncu_batched_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 \
   -o gpurun_out/c3pass1_$TAG python scripts/p1_time.py --data illcond --eps 1e-12 --reps 2 > gpurun_out/ncu_c3_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact -s 1 -c 1 \
   -o gpurun_out/exact_$TAG python scripts/exact_time.py > gpurun_out/ncu_exact_$TAG.log 2>&1
timeout 300 python scripts/exact_time.py > gpurun_out/exact_time_$TAG.json 2>&1
timeout 300 python scripts/latency.py > gpurun_out/latency_$TAG.jsonl 2>&1
timeout 300 python scripts/solver_bench.py > gpurun_out/solver_bench_$TAG.jsonl 2>&1
timeout 300 python scripts/spmv_time.py > gpurun_out/spmv_time_$TAG.jsonl 2>&1
timeout 300 python scripts/sustained_probe.py > gpurun_out/sustained_probe_$TAG.jsonl 2>&1
( for n in 10000 1000000 268435456; do timeout 120 python scripts/step_graph_time.py $n; done ) > gpurun_out/step_graph_$TAG.jsonl 2>&1
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke_$TAG.log 2>&1
timeout 600 bash scripts/check_multirank.sh > gpurun_out/multirank_$TAG.log 2>&1
# summarise every capture here (ncu is on the box) and keep only the reports named in KEEP
# (gpurun copies back at most 64 MiB)
for rep in pass1 batched c3pass1 exact; do
  [ -f gpurun_out/${rep}_$TAG.ncu-rep ] && python tools/ncu_summary.py gpurun_out/${rep}_$TAG.ncu-rep gpurun_out/${rep}_${TAG}_ncu > /dev/null 2>&1
  case " ${KEEP:-batched} " in *" $rep "*) ;; *) rm -f gpurun_out/${rep}_$TAG.ncu-rep ;; esac
done
[ -f gpurun_out/launches_$TAG.csv ] && python tools/ncu_summary.py --launches gpurun_out/launches_$TAG.csv gpurun_out/launches_$TAG > /dev/null 2>&1
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/bench_$TAG.json gpurun_out/exact_time_$TAG.json
echo done
