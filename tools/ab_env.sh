# experiments build under several env settings (early window, --skip 0), alternating
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]/64*1000,2), "us")'
for i in 1 2; do
  for e in "$@"; do
    echo -n "$e : "; env $e FADE_LIB_PATH=$PWD/build/exp/libfade_b200.so python bench.py --skip 0 --no-sweep --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | python -c "$P"
  done
done
