#!/usr/bin/env bash
# GPU suite + smoke + default bench (no CPU legs); logs under gpurun_out/<tag>_*
cd "$(dirname "$0")/.."
tag=${1:-run}
mkdir -p gpurun_out
timeout 900 python -u -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/${tag}_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_gpu_tests.txt
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.txt
timeout 400 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -3 gpurun_out/${tag}_gpu_tests.txt; tail -2 gpurun_out/${tag}_smoke.txt; grep -o '"value": [0-9.]*, "unit": "pairs/s", "n_gpus[^,]*\|"ms_per_step": [0-9.]*\|correct_offsets": "[^"]*\|"clocks": {[^}]*}' gpurun_out/${tag}_bench.json
