timeout 150 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | grep -E "passed|failed|Error|assert|Timeout" | head -8
timeout 120 python bench.py --mode fused --steps 50 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value", d["value"], "ms", d["ms_per_step"], d["config"]["correct_offsets"])'
timeout 120 python tools/pipe_trace.py 2>&1 | sed -n '5,45p' | awk 'NR%3==1'
