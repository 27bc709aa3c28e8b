"""Canonical FP64 work model of the path and the
measured B200 FP64 peak, shared by bench.py and the run records.

Per box with n rows, s probes, rank r (2 flops per madd), in the canonical
Householder realisation of Alg. 2 -- extra work a kernel does is never
credited:
  probe QR            2 n^2 (s - n/3)            (x2 sides)
  apply Q + solve     4 n^2 s - 2 n^3 + n^3      (x2 sides)
  col() basis QR      4 r^2 (n - r/3)            (x2 sides)
  discrepancy         12 r n^2
  lift                4 n^2 s + 8 r n s
  root                2 n^2 (s - n/3) + 4 n^2 s - n^3,  n = 2r
"""

import numpy as np

# profiles/fp64_peaks_r02.json: best DMMA m8n8k4 / m16n8k4 rate on this pool's
# B200 at 1965 MHz (no throttle reasons); NVIDIA's spec figure is 40 TF/s.
FP64_PEAK_TFLOPS = 37.03
FP64_SPEC_TFLOPS = 40.0

PHASES = ("probe_qr", "panel_factors", "apply_q_solve", "basis_qr", "discrepancy_gemm", "lift_gemm")


def canonical_phase_flops(n, s, r):
    return {
        "probe_qr": 2 * (2 * n * n * (s - n / 3)),
        "panel_factors": 0.0,
        "apply_q_solve": 2 * ((4 * n * n * s - 2 * n ** 3) + n ** 3),
        "basis_qr": 2 * (4 * r * r * (n - r / 3)),
        "discrepancy_gemm": 12 * r * n * n,
        "lift_gemm": 4 * n * n * s + 8 * r * n * s,
    }


def canonical_total_flops(tree, s, r, top_level=1):
    """Whole sweep (levels depth..top_level, plus the root when top_level == 1)."""
    total = 0.0
    for level in range(tree.depth, top_level - 1, -1):
        sizes = tree.level_sizes(level) if level == tree.depth else np.full(1 << level, 2 * r)
        for n in np.unique(sizes):
            total += int((sizes == n).sum()) * sum(canonical_phase_flops(int(n), s, r).values())
    if top_level == 1:
        n = 2 * r
        total += 2 * n * n * (s - n / 3) + 4 * n * n * s - n ** 3
    return total
