# this tree's bench.py (early window, --skip 0) over the libraries of several
# commits (build/bis/<commit>; same ABI since 9b10a19), alternating on one box
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]/64*1000,2), "us")'
for i in 1 2 3; do
  for c in "$@"; do
    if [ "$c" = HEAD ]; then L=$PWD/paper_2604_07239_b200/_lib/libfade_b200.so; else L=$PWD/build/bis/$c/paper_2604_07239_b200/_lib/libfade_b200.so; fi
    echo -n "$c : "; FADE_LIB_PATH=$L python bench.py --skip 0 --no-sweep --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$P"
  done
done
