"""Summarise an ncu --csv metrics log of tools/profile_step.py (the last
timestep's launches) into one row per kernel: time, tensor-pipe activity,
DRAM / L2 bytes and throughput.

    python tools/ncu_table.py launches.csv [--steps N]
"""
import collections
import csv
import sys

NAMES = [  # launch order of one timestep (engine.cu forward() / backward())
    "trunk_fwd", "gemm route+W_mem (split-K)", "mix_fwd", "gemm down", "bmm_fwd",
    "gemm up+cgate", "coarse_fwd", "gemm e12+GeGLU (persistent, pairs)", "gemm F (pairs, split-K)",
    "out_fwd", "gemm head", "head", "head_quant (coder stream)", "encode (coder stream)",
    "gemm dh", "out_bwd", "gemm dwide+GeGLU-bwd (pairs)", "gemm dz2 (pairs, split-K)",
    "gemm dW12+Adam (side, pairs)", "coarse_bwd", "gemm dW_f+dW_head+Adam (side)", "gemm du+dhm_c",
    "bmm_bwd+W_U Adam", "gemm dz", "gemm dW_up/cgate/down+Adam (side)", "mix_bwd",
    "gemm dx_r+dblock", "gemm dW_route+dW_mem+Adam (side)", "trunk_bwd", "small_adam"]


def load(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault(r[ii], {"k": r[ki]})[r[mi]] = r[vi]
    return list(d.values())


def main():
    items = load(sys.argv[1])
    # profile_step runs a few timesteps: take the last, from its trunk_fwd
    starts = [i for i, it in enumerate(items) if "k_trunk_fwd" in it["k"]]
    step = items[starts[-1]:]
    f = lambda it, k: float(it.get(k, "nan").replace(",", ""))
    tot = sum(f(it, "gpu__time_duration.sum") for it in step) / 1e3
    print(f"{'#':>2} {'kernel':38s} {'us':>6} {'share':>6} {'tensor%':>7} {'dram%':>6} "
          f"{'DRAM MB':>8} {'GB/s':>6} {'L2 MB':>7}")
    for i, it in enumerate(step):
        us = f(it, "gpu__time_duration.sum") / 1e3
        mb = (f(it, "dram__bytes_read.sum") + f(it, "dram__bytes_write.sum")) / 1e6
        name = NAMES[i] if len(step) == len(NAMES) else it["k"][:38]
        print(f"{i:2d} {name[:38]:38s} {us:6.1f} {us / tot:6.1%} "
              f"{f(it, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):7.1f} "
              f"{f(it, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} {mb:8.1f} "
              f"{mb / us * 1e3:6.0f} {f(it, 'lts__t_bytes.sum') / 1e6:7.1f}")
    print(f"   sum (serialised, cold caches) {tot:.1f} us")


if __name__ == "__main__":
    main()
