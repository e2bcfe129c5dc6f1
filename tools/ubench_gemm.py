"""Standalone timing of the binary32 trailing update (mpirg_ubench_gemm_f32)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2311_14616_b200 import lib
    L = lib()
    tf, ms = C.c_double(), C.c_double()
    L.mpirg_ffma_peak(C.byref(tf), C.byref(ms))
    peak = tf.value
    print(f"ffma peak {peak:.1f} TFLOP/s")
    cases = [(16384, 128, 128), (16384, 64, 128), (16384, 128, 64), (8192, 128, 128),
             (4096, 128, 0), (4096, 64, 0)]
    if len(sys.argv) > 1:
        cases = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
    for n, k, tile in cases:
        rc = L.mpirg_ubench_gemm_f32(n, k, tile, 5, C.byref(tf), C.byref(ms))
        bytes_c = 8.0 * (n - k) ** 2
        print(f"n={n} K={k} tile={tile} rc={rc} {ms.value:.3f} ms {tf.value:.1f} TFLOP/s "
              f"({tf.value / peak * 100:.0f}% FFMA) C-traffic {bytes_c / ms.value / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
