# steady-state (default --skip) and early window of several libraries
# (build/bis/<name>, or HEAD = this tree's), alternating on one box
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]/64*1000,2), "us steady", round(d["config"]["early_window_ms_per_step"]/64*1000,2), "us early")'
for i in 1 2; do
  for c in "$@"; do
    if [ "$c" = HEAD ]; then L=$PWD/paper_2604_07239_b200/_lib/libfade_b200.so; else L=$PWD/build/bis/$c/paper_2604_07239_b200/_lib/libfade_b200.so; fi
    echo -n "$c : "; FADE_LIB_PATH=$L python bench.py --no-sweep --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | python -c "$P"
  done
done
