#!/bin/bash
# usage: tools/bench_variants.sh name1 name2 ...   (main = the in-tree library)
for v in "$@"; do
  if [ "$v" = main ]; then L=; else L=paper_1302_3120_b200/variants/libcssar_$v.so; fi
  CSSAR_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 100 --warmup 10 ${BENCH_ARGS} 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})" \
    || echo "$v FAILED"
done
