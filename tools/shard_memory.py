"""Per-rank HBM estimate of the ghost-row sharded store.

A vertex of expected degree λ (Chung-Lu weights w_i ∝ i^-α, mean degree m/n) has an
out-edge into a given one of P shards with probability 1 - exp(-λ/P); ghosts = non-owned
vertices with such an edge.  Prints the table rows of DESIGN.md §6."""
import numpy as np


def ghost_fraction(P, mean_deg, alpha=0.8):
    x = np.linspace(1e-7, 1, 2_000_001)
    lam = mean_deg * (1 - alpha) * x ** -alpha
    return 1 - np.trapezoid(np.exp(-lam / P), x)


def plan(name, n, m, dims, P, headroom=0.10, chunk=1 << 22):
    own = n / P
    f = ghost_fraction(P, m / n)
    loc = own + (n - own) * f
    cap = loc * (1 + headroom)
    L = len(dims) - 1
    row = max(dims) * 4
    inputs = L * cap * row
    delta = cap * row
    owned = (L + 2) * own * row  # S^0..S^{L-1}, final H, update image
    e = m / P
    graph = e * 16 * 1.25 + cap * 16 * 2
    maps = n * 4 + cap * 16 + L * cap * 16
    xch = 2 * chunk * (row + 4)
    tot = inputs + delta + owned + graph + maps + xch
    gb = 1e9
    print(f"{name}: P={P} ghost fraction {f:.3f}, owned {own/1e6:.2f}M, local {loc/1e6:.1f}M, cap {cap/1e6:.1f}M")
    print(f"  inputs {inputs/gb:.1f} GB, delta {delta/gb:.1f}, owned {owned/gb:.1f}, graph {graph/gb:.1f}, "
          f"maps+frontier {maps/gb:.1f}, exchange {xch/gb:.1f} -> total {tot/gb:.1f} GB")


if __name__ == "__main__":
    plan("configs[4] C5 GCN-2L", 111.06e6, 1.616e9, [128, 128, 128], 8)
    plan("configs[3] C4 GIN-3L", 10e6, 500e6, [128, 128, 128, 128], 8)
    plan("configs[3] C4 GIN-3L", 10e6, 500e6, [128, 128, 128, 128], 2)
