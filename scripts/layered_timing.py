"""Train-only step time of the layered path (K=50, R=120, S=10, 4 layers)
at the Fig. 6 widths, and of VM_LAYERED=1 at hidden 32/128 against the fused
kernels (run twice: with and without VM_LAYERED=1)."""
import sys

sys.path.insert(0, ".")
from paper_2302_01838_b200.trainer import benchmark  # noqa: E402

for r in benchmark([50], [int(h) for h in (sys.argv[1:] or ["32", "128", "256", "512", "1024"])],
                   timed_steps=10, warmup_steps=3, modes=("vectorised",)):
    h = r.hidden
    flop = 6.0 * 1200 * (33 * h + 2 * h * h + 4 * h) * r.k
    print(f"K={r.k} h={h}: {r.ms:.3f} ms  {flop / (r.ms * 1e-3) / 1e12:.1f} TFLOP/s", flush=True)
