#!/bin/bash
# Round evidence: smoke, GPU tests (incl. slow), bench, launch list, ncu full of pass1.
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 1100 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 500 --warmup 10 --e2e-steps 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 \
   -o gpurun_out/pass1_$TAG python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_pass1_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_score|k_finalize" -s 2 -c 2 \
   -o gpurun_out/small_$TAG python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_small_$TAG.log 2>&1
echo done
