# round-1 build (build/r1tree, its own bench.py: first K steps after warm-up)
# vs this tree with --skip 0 (the same early window), alternating on one box
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]/64*1000,2), "us", round(d["value"],4))'
for i in 1 2; do
  echo -n "r1 : "; (cd build/r1tree && python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$P")
  echo -n "now: "; python bench.py --skip 0 --no-sweep --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$P"
done
