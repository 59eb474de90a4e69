# B=512 early-window timestep of several builds (each a tree under build/bis/<commit>
# with its own bench.py), alternating on one box
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]/64*1000,2), "us")'
run() {
  (cd "$1" && { python bench.py --skip 0 --no-sweep --no-cpu-baseline --no-e2e 2>/dev/null \
     || python bench.py --no-sweep --no-cpu-baseline --no-e2e 2>/dev/null \
     || python bench.py --no-cpu-baseline --no-e2e 2>/dev/null; } | python -c "$P")
}
for i in 1 2; do
  echo -n "r1      : "; run build/r1tree
  for c in "$@"; do echo -n "$c : "; run build/bis/$c; done
  echo -n "HEAD    : "; run .
done
