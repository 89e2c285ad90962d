for pr in 0 1 2; do echo "== probe $pr"; MTB_PIPE_PROBE=$pr python tools/pipe_trace.py 2>&1 | sed -n '1,4p;14,22p' | grep -v "^step ms 5\|^step ms 3"; done
