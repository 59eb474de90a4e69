"""Per-GEMM tensor-pipe / memory summary of an `ncu --set full` report of the
tcgen05 GEMMs of one timestep (tools/profile_step.py), for profiles/.

    python tools/ncu_gemms.py report.ncu-rep [batch]
"""
import csv
import subprocess
import sys

M = ("gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum,"
     "lts__t_sectors.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,"
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
NAMES = ["route+W_mem fwd (split-K 17+2)", "down fwd (split-K)", "up+cgate fwd (split-K)",
         "F fwd (pairs, split-K 18)", "head fwd (split-K)", "dh", "dwide+GeGLU-bwd (pairs)",
         "dz2 (pairs, split-K 18)", "dW12+Adam (pairs, 2/SM)", "dW_f+dW_head+Adam", "du+dhm_c", "dz",
         "dW_up/cgate/down+Adam", "dx_r+dblock", "dW_route+dW_mem+Adam"]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "usecond": 1.0, "nsecond": 1e-3,
         "msecond": 1e3}


def flops(B, H=512, X=128, E=8192, C=4096):
    return [2 * B * H * (H + C), 2 * B * X * H, 2 * B * H * (X + H), 2 * B * H * E, 2 * B * 256 * H,
            2 * B * H * 256, 2 * B * E * H, 2 * B * H * 2 * E, 2 * B * H * 2 * E,
            2 * B * (E * H + H * 256), 2 * B * (H * X + H * H), 2 * B * X * H,
            2 * B * (X * H + H * H + H * X), 2 * B * H * (H + 32), 2 * B * H * (H + C)]


def main():
    rep = sys.argv[1]
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", M],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}

    def g(r, k):
        return float(r[ix[k]].replace(",", "")) * SCALE.get(units[ix[k]], 1.0)

    print(f"tcgen05 kind::tf32 GEMMs of one B = {B} timestep: ncu --set full --clock-control none")
    print("(cold caches, serialised; pipe% = sm__pipe_tensor_cycles_active % of peak, "
          "100% ~ 1.1 PF/s dense TF32; TF/s = algorithmic FLOPs / duration)")
    print(f"{'GEMM':34s} {'grid':>5} {'us':>6} {'pipe%':>6} {'TF/s':>6} {'dram%':>6} "
          f"{'DRAM MB':>8} {'L2 MB':>7}")
    for n, f, r in zip(NAMES, flops(B), rows[2:]):
        us = g(r, "gpu__time_duration.sum")
        mb = g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum")
        print(f"{n:34s} {r[ix['launch__grid_size']]:>5} {us:6.1f} "
              f"{g(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{f / us / 1e6:6.0f} {g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{mb:8.1f} {g(r, "lts__t_sectors.sum") * 32e-6:7.1f}")


if __name__ == "__main__":
    main()
