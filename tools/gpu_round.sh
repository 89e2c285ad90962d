#!/usr/bin/env bash
# GPU suite + smoke + benches; logs under gpurun_out/<tag>_*.  Usage: gpu_round.sh TAG [tests|bench|all]
cd "$(dirname "$0")/.."
tag=${1:-run}; what=${2:-all}
mkdir -p gpurun_out
if [ "$what" = tests ] || [ "$what" = all ]; then
  timeout 1500 python -u -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfEs > gpurun_out/${tag}_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_gpu_tests.txt
  timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.txt
  tail -15 gpurun_out/${tag}_gpu_tests.txt; tail -2 gpurun_out/${tag}_smoke.txt
fi
if [ "$what" = bench ] || [ "$what" = all ]; then
  timeout 600 python bench.py --steps 40 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
  echo "bench rc=$?"; tail -c 3000 gpurun_out/${tag}_bench.json
  for c in 1 3 4; do
    timeout 400 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/${tag}_bench_c$c.json 2> gpurun_out/${tag}_bench_c$c.err
    echo "config $c rc=$?"; grep -o '"value": [0-9.]*, "unit": "pairs/s", "n_gpus[^,]*\|"ms_per_step": [0-9.]*\|correct_offsets": "[^"]*\|"oracle_match": {[^}]*}' gpurun_out/${tag}_bench_c$c.json
  done
fi
