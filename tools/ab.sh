#!/usr/bin/env bash
# Same-box A/B: current library vs _lib/exp/$1.so, alternating bench runs.  Usage: tools/ab.sh NAME [bench args]
cd "$(dirname "$0")/.."
name=$1; shift
L=$PWD/paper_2007_06483_b200/_lib/exp/$name.so
for i in 1 2 3; do
  for v in cur $name; do
    if [ $v = cur ]; then unset MTB_LIB_PATH; else export MTB_LIB_PATH=$L; fi
    r=$(timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-oracle-check "$@" 2>/dev/null | grep -o '"value": [0-9.]*' | head -1)
    echo "$v $r"
  done
done
unset MTB_LIB_PATH
