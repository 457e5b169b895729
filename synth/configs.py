"""The five workloads of BASELINE.json ``configs`` as plain data.

Physical constants follow the config text: mu_s' = 10 /cm, background
mu_a = 0.05 /cm, anomaly mu_a = 0.15 /cm, nu = 2.2e10 cm/s, D = 1/(3(mu_a+mu_s'))
evaluated with the background mu_a (reading R4).  Frequencies are
modulation frequencies f in Hz; the PDE uses omega = 2*pi*f (Eq. (2.1),
"i omega / nu").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

MHZ = 1.0e6


@dataclass(frozen=True)
class DOTConfig:
    name: str
    n: Tuple[int, int, int]            # interior FD nodes (nx, ny, nz)
    L: Tuple[float, float, float]      # domain extents (cm): [0,Lx]x[0,Ly]x[0,Lz]
    freqs_hz: Tuple[float, ...]        # modulation frequencies f (omega = 2 pi f)
    src_grid: Tuple[int, int]          # point sources: (n_ax, n_ay) array on top face z=0
    det_grid: Tuple[int, int]          # point detectors: array on bottom face z=Lz
    n_rbf: int                         # PaLS basis functions of the current iterate p
    n_rbf_true: int = 2                # hidden "true" level set used for the data
    ls: Optional[int] = None           # simultaneous sources (None: W = I)
    ld: Optional[int] = None           # simultaneous detectors (None: V = I)
    n_opt: int = 0                     # optimized directions (config 3)
    n_subspace_iters: int = 0          # subspace iterations for the optimized directions
    seed: int = 0                      # seed of p, p_true and noise
    sketch_seed: int = 1               # seed of the Rademacher W, V
    mus_prime: float = 10.0
    mua_bg: float = 0.05
    mua_anom: float = 0.15
    nu: float = 2.2e10                 # speed of light in the medium, cm/s
    gamma: float = 1.0e-2              # ||x||^dagger regulariser (Sec. 2)
    eps: float = 0.1                   # smoothed-Heaviside width
    cutoff: float = 0.15               # level-set cut-off c (Fig. 1 caption)
    noise: float = 0.01                # relative Gaussian data noise
    note: str = field(default="", compare=False)

    @property
    def n_s(self) -> int:
        return self.src_grid[0] * self.src_grid[1]

    @property
    def n_d(self) -> int:
        return self.det_grid[0] * self.det_grid[1]

    @property
    def n_p(self) -> int:
        return 5 * self.n_rbf

    @property
    def n_freq(self) -> int:
        return len(self.freqs_hz)

    @property
    def N(self) -> int:
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def D(self) -> float:
        return 1.0 / (3.0 * (self.mua_bg + self.mus_prime))

    def with_(self, **kw) -> "DOTConfig":
        d = {k: getattr(self, k) for k in self.__dataclass_fields__}
        d.update(kw)
        return DOTConfig(**d)


FREQS3 = (0.0, 70 * MHZ, 140 * MHZ)
FREQS5 = (0.0, 50 * MHZ, 100 * MHZ, 150 * MHZ, 200 * MHZ)

CONFIGS = (
    DOTConfig(name="tiny16", n=(16, 16, 16), L=(4.0, 4.0, 4.0), freqs_hz=(0.0,),
              src_grid=(4, 4), det_grid=(4, 4), n_rbf=4, seed=0,
              note="configs[0]: tiny DOT forward + Jacobian, full W=V=I"),
    DOTConfig(name="sketch32", n=(32, 32, 32), L=(8.0, 8.0, 8.0), freqs_hz=FREQS3,
              src_grid=(8, 8), det_grid=(8, 8), n_rbf=8, ls=8, ld=8, seed=0, sketch_seed=1,
              note="configs[1]: 64 src/det, 3 freqs, Rademacher W,V 64x8"),
    DOTConfig(name="full64", n=(64, 64, 64), L=(8.0, 8.0, 8.0), freqs_hz=FREQS3,
              src_grid=(16, 16), det_grid=(16, 16), n_rbf=16, ls=12, ld=12, seed=0, sketch_seed=1,
              note="configs[2]: full-data 256+256 RHS/freq + sketched Jacobian W,V 256x12"),
    DOTConfig(name="opt96", n=(96, 96, 96), L=(8.0, 8.0, 8.0), freqs_hz=FREQS5,
              src_grid=(32, 32), det_grid=(32, 32), n_rbf=24, ls=12, ld=12, n_opt=2,
              n_subspace_iters=5, seed=0, sketch_seed=1,
              note="configs[3]: 10 Rademacher + 2 optimized directions"),
    DOTConfig(name="all128", n=(128, 128, 128), L=(8.0, 8.0, 8.0), freqs_hz=FREQS5,
              src_grid=(32, 32), det_grid=(32, 32), n_rbf=32, seed=0,
              note="configs[4]: all sources/detectors, full Jacobian, RHS-sharded"),
)


def config_by_name(name: str) -> DOTConfig:
    for c in CONFIGS:
        if c.name == name:
            return c
    raise KeyError(name)
