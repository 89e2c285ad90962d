# parity tests + short bench (no cpu baseline / e2e)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>&1 | tail -2
