"""Test helpers: bridge oracle weights to the product, comparisons."""

from __future__ import annotations

import numpy as np

import oracle
from oracle.model import OracleConfig


def product_config(ocfg: OracleConfig):
    from paper_2507_11830_b200.config import ModelConfig
    return ModelConfig(n_layers=ocfg.n_layers, n_heads=ocfg.n_heads, head_dim=ocfg.head_dim,
                       ffn_dim=ocfg.ffn_dim, vocab_size=ocfg.vocab_size, max_seq=ocfg.max_seq,
                       n_kv_heads=ocfg.n_kv_heads, pos=ocfg.pos, mlp=ocfg.mlp,
                       norm_eps=ocfg.norm_eps, rope_theta=ocfg.rope_theta,
                       rope_scaling=ocfg.rope_scaling).validate()


def host_dict(ow) -> dict:
    return {"embed": ow.embed, "layers": ow.layers, "final_gain": ow.final_gain, "head": ow.head,
            "seed": ow.seed}


def device_weights(ow, world_size: int):
    from paper_2507_11830_b200.weights import ModelWeights
    return ModelWeights.from_host(product_config(ow.config), host_dict(ow), world_size)


def rel_err(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30))


def top2_margin(row) -> float:
    s = np.sort(np.asarray(row, dtype=np.float64))
    return float(s[-1] - s[-2])


def c1_prompts():
    rng = np.random.default_rng(7)
    lens = [int(x) for x in rng.integers(32, 129, size=8)]
    return [[int(t) for t in rng.integers(0, 256, size=n)] for n in lens]
