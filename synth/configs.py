"""The five workload configurations C1..C5 (SURVEY.md §8 table, §8(d) recipes).

Values come from BASELINE.json ``configs`` first and from the paper's
Supp. Table 5 / P:957 where BASELINE.json is silent.
Non-paper choices are marked and listed in DESIGN.md ("readings").
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict
from typing import Tuple


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    stand_in_for: str
    sizes: Tuple[int, ...]          # n_1 .. n_L (paper notation, input first)
    epsilon: float                  # ER density parameter
    alpha: float                    # All-ReLU slope (Eq. 3)
    activation: str = "all_relu"    # "all_relu" | "relu"
    dropout: float = 0.0            # inverted dropout rate on hidden activations
    init: str = "he_uniform"        # "normal" | "xavier" | "he_uniform" (Table 5)
    batch: int = 128                # per-rank minibatch B
    lr: float = 0.01                # eta
    momentum: float = 0.9           # mu
    weight_decay: float = 2e-4      # lambda: value not given by the paper (non-paper default)
    zeta: float = 0.3               # SET prune fraction
    n_samples: int = 2000
    epochs: int = 3
    prune: bool = False             # Importance Pruning (Alg. 2)
    prune_percentile: float = 5.0   # rho (Supp. C)
    prune_every: int = 1            # p
    prune_start: int = 0            # tau (paper: 200; C3 uses 0 so it fires in short runs)
    binary_input: bool = False      # inputs in {0, 1}, Bernoulli(0.05), stored fp32 (C5 and the Table 4 rows)
    data_seed: int = 0
    model_seed: int = 0

    @property
    def n_layers(self) -> int:
        return len(self.sizes)

    @property
    def n_classes(self) -> int:
        return self.sizes[-1]

    def to_json(self) -> dict:
        d = asdict(self)
        d["sizes"] = list(self.sizes)
        return d


def _cfg(idx: int, **kw) -> WorkloadConfig:
    return WorkloadConfig(data_seed=1000 + idx, model_seed=2000 + idx, **kw)


CONFIGS = {
    # BASELINE.json configs[0]; Madelon stand-in
    "C1": _cfg(1, name="C1", stand_in_for="Madelon (PAPER.md:147)",
               sizes=(500, 400, 100, 400, 2), epsilon=10.0, alpha=0.6,
               dropout=0.0, init="he_uniform", batch=128, lr=0.01,
               n_samples=2000, epochs=3),
    # configs[1]; FashionMNIST stand-in
    "C2": _cfg(2, name="C2", stand_in_for="FashionMNIST (PAPER.md:148)",
               sizes=(784, 1000, 1000, 1000, 10), epsilon=20.0, alpha=0.75,
               dropout=0.3, init="he_uniform", batch=128, lr=0.01,
               n_samples=60000, epochs=1),
    # configs[2]; Leukemia stand-in, importance pruning each epoch
    "C3": _cfg(3, name="C3", stand_in_for="Leukemia GSE13159 (PAPER.md:145)",
               sizes=(54675, 27500, 27500, 18), epsilon=10.0, alpha=0.75,
               dropout=0.3, init="normal", batch=5, lr=0.005,
               n_samples=2096, epochs=1, prune=True, prune_percentile=5.0,
               prune_every=1, prune_start=0),
    # configs[3]; HIGGS x100 stand-in
    "C4": _cfg(4, name="C4", stand_in_for="HIGGS x100 (PAPER.md:146)",
               sizes=(28, 1000, 1000, 1000, 2), epsilon=10.0, alpha=0.05,
               dropout=0.3, init="xavier", batch=128, lr=0.01,
               n_samples=10_500_000, epochs=1),
    # configs[4]; Table 4 row 1 scaled up
    "C5": _cfg(5, name="C5", stand_in_for="make_classification 65536-feature set (PAPER.md:409)",
               sizes=(65536, 500000, 500000, 500000, 2), epsilon=20.0, alpha=0.5,
               dropout=0.0, init="he_uniform", batch=128, lr=0.01,
               n_samples=100_000, epochs=1, binary_input=True),
}

# Width scaling: the five architectures of the paper's Table 4
# ("65536-5M x 4-2" = four hidden layers of 5M neurons), trained there on a
# 10000 x 65536 make_classification set, 70% train, batch 128, lr 0.01, momentum
# 0.9, dropout 0.4.  Stand-in data: the C5 binary recipe (Bernoulli(0.05) features, linear
# teacher), 7000 training rows.  alpha / init / weight decay as C5 (the paper gives none for them).
_T4_ROWS = {
    "T1": ((65536, 500_000, 500_000, 2), 10.0),
    "T2": ((65536, 2_500_000, 2_500_000, 2), 5.0),
    "T3": ((65536, 5_000_000, 5_000_000, 2), 5.0),
    "T4": ((65536,) + (5_000_000,) * 4 + (2,), 1.0),
    "T5": ((65536,) + (5_000_000,) * 10 + (2,), 1.0),
}
for _k, (_name, (_sizes, _eps)) in enumerate(_T4_ROWS.items()):
    CONFIGS[_name] = _cfg(10 + _k, name=_name, stand_in_for=f"Table 4 row {_k + 1} (PAPER.md:426-434), "
                          "make_classification 65536-feature set (PAPER.md:409)",
                          sizes=_sizes, epsilon=_eps, alpha=0.5, dropout=0.4, init="he_uniform", batch=128,
                          lr=0.01, n_samples=7000, epochs=1, binary_input=True)


def get_config(name: str, **overrides) -> WorkloadConfig:
    base = CONFIGS[name]
    if not overrides:
        return base
    d = base.to_json()
    d.update(overrides)
    d["sizes"] = tuple(d["sizes"])
    return WorkloadConfig(**d)
