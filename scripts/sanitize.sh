#!/bin/bash
# compute-sanitizer over smoke() and a small slice of every GPU test file:
# memcheck (out-of-bounds / misaligned / leaks of device memory), racecheck
# and synccheck (shared-memory hazards in pass1 / batched / exact). Outputs
# the summaries under gpurun_out/sanitize/.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/sanitize; mkdir -p $O
CS="compute-sanitizer --target-processes all --print-limit 20"
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
ids() {  # file regex -> node ids (collected on the box; GPU tests skip at import elsewhere)
  python -m pytest -q --collect-only "$1" 2>/dev/null | grep '::' | grep -E "$2"
}
P_MEM=$(ids tests/test_gpu_parity.py 'toy|empty|errors|graph_one_call|pass2_over_cold|c_abi_dot_host\[(0|1000)-|random_against_oracle\[(auto|lean-wide-queue|full-queue)-(exact|ranged:3|split:4)-[01]\]|golden_case\[auto-')
P_RACE=$(ids tests/test_gpu_parity.py 'toy|random_against_oracle\[(auto|full|lean-wide)-(exact|ranged:3)-0\]')
echo "parity memcheck: $(echo $P_MEM | wc -w) tests; racecheck: $(echo $P_RACE | wc -w)"
run() {  # name tool cmd...
  local name=$1 tool=$2; shift 2
  timeout 600 $CS --tool $tool "$@" > $O/$name.$tool.log 2>&1
  echo "$name $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/$name.$tool.log | tail -1)"
}
run smoke memcheck python -c "import __graft_entry__ as g; g.smoke()"
run parity memcheck python -m pytest -q -x $P_MEM
run batched memcheck python -m pytest -q -x tests/test_gpu_batched.py -k "not c4"
run exact memcheck python -m pytest -q -x tests/test_gpu_exact.py -k "not c2"
run apps memcheck python -m pytest -q -x tests/test_gpu_apps.py -k "spmv or vector or eager"
run smoke racecheck python -c "import __graft_entry__ as g; g.smoke()"
run smoke synccheck python -c "import __graft_entry__ as g; g.smoke()"
run parity racecheck python -m pytest -q -x $P_RACE
run batched racecheck python -m pytest -q -x tests/test_gpu_batched.py -k "not c4"
run exact racecheck python -m pytest -q -x tests/test_gpu_exact.py -k "not c2"
