"""OPT decoder geometry and random-init weights resident in HBM.

The reference has no decoder (SURVEY.md §8a note 2); the layer semantics
follow transformers' modeling_opt (pre-LN, biases on all projections,
learned positions with offset 2, tied LM head).  Weights are synthetic
(no network for checkpoints): normal(0, std) for every Linear weight AND
bias, LN gamma = 1 + N(0, std), beta = N(0, std), embeddings N(0, emb_std)
(SURVEY.md §8d), generated with a seeded torch generator directly on the
target device and stored fp16 in the PyTorch [out, in] layout the tcgen05
GEMM consumes (K-major).  q/k/v are fused into one [3h, h] matrix so the
rows [h, 3h) are the [W_k | W_v] operand of the recompute GEMM K1.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .costmodel import ModelSpec


@dataclass(frozen=True)
class OPTConfig:
    hidden: int
    layers: int
    heads: int
    ffn: int
    vocab: int = 50272
    max_pos: int = 2048
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def spec(self) -> ModelSpec:
        return ModelSpec(hidden_dim=self.hidden, num_layers=self.layers, num_heads=self.heads, ffn_dim=self.ffn,
                         precision_bytes=2)

    def describe(self) -> str:
        return (f"OPT decoder h{self.hidden} x{self.layers} layers, {self.heads} heads, ffn {self.ffn}, "
                f"vocab {self.vocab} (random init)")

    def with_positions(self, n: int) -> "OPTConfig":
        """Synthetic learned-position table long enough for n positions (config 5 sweeps past 2048)."""
        return OPTConfig(self.hidden, self.layers, self.heads, self.ffn, self.vocab, max(self.max_pos, n), self.eps)


PRESETS = {
    "opt-125m": OPTConfig(hidden=768, layers=12, heads=12, ffn=3072),
    "opt-6.7b": OPTConfig(hidden=4096, layers=32, heads=32, ffn=16384),
    "opt-13b": OPTConfig(hidden=5120, layers=40, heads=40, ffn=20480),
    "opt-30b": OPTConfig(hidden=7168, layers=48, heads=56, ffn=28672),
}


def preset(name: str) -> OPTConfig:
    key = name.strip().lower()
    if key not in PRESETS:
        raise ValueError(f"unknown model {name!r}; known: {', '.join(sorted(PRESETS))}")
    return PRESETS[key]


@dataclass
class LayerWeights:
    ln1_g: torch.Tensor
    ln1_b: torch.Tensor
    wqkv: torch.Tensor  # [3h, h]
    bqkv: torch.Tensor  # [3h]
    wo: torch.Tensor    # [h, h]
    bo: torch.Tensor
    ln2_g: torch.Tensor
    ln2_b: torch.Tensor
    w1: torch.Tensor    # [ffn, h]
    b1: torch.Tensor
    w2: torch.Tensor    # [h, ffn]
    b2: torch.Tensor

    @property
    def w_kv(self) -> torch.Tensor:
        """[2h, h] view = rows of W_k then W_v (the K1 operand)."""
        h = self.wqkv.shape[1]
        return self.wqkv[h:]

    @property
    def b_kv(self) -> torch.Tensor:
        h = self.wqkv.shape[1]
        return self.bqkv[h:]


@dataclass
class OPTWeights:
    cfg: OPTConfig
    layers: list[LayerWeights]
    embed: torch.Tensor  # [V, h] (tied LM head)
    pos: torch.Tensor    # [max_pos + 2, h]
    lnf_g: torch.Tensor
    lnf_b: torch.Tensor
    meta: dict = field(default_factory=dict)

    @classmethod
    def random(cls, cfg: OPTConfig, seed: int = 0, device: str | torch.device = "cuda", std: float = 0.02,
               emb_std: float | None = None) -> "OPTWeights":
        dev = torch.device(device)
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        emb_std = std if emb_std is None else emb_std

        def rnd(*shape, s=std, base=0.0):
            t = torch.empty(*shape, device=dev, dtype=torch.float32)
            t.normal_(0.0, s, generator=g)
            if base:
                t += base
            return t.to(torch.float16)

        h, f = cfg.hidden, cfg.ffn
        layers = []
        for _ in range(cfg.layers):
            layers.append(LayerWeights(
                ln1_g=rnd(h, base=1.0), ln1_b=rnd(h),
                wqkv=rnd(3 * h, h), bqkv=rnd(3 * h),
                wo=rnd(h, h), bo=rnd(h),
                ln2_g=rnd(h, base=1.0), ln2_b=rnd(h),
                w1=rnd(f, h), b1=rnd(f),
                w2=rnd(h, f), b2=rnd(h),
            ))
        return cls(cfg=cfg, layers=layers, embed=rnd(cfg.vocab, h, s=emb_std), pos=rnd(cfg.max_pos + 2, h, s=emb_std),
                   lnf_g=rnd(h, base=1.0), lnf_b=rnd(h), meta={"seed": seed, "std": std, "emb_std": emb_std})

    def to(self, device) -> "OPTWeights":
        mv = lambda t: t.to(device)  # noqa: E731
        return OPTWeights(
            cfg=self.cfg,
            layers=[LayerWeights(**{k: mv(getattr(lw, k)) for k in lw.__dataclass_fields__}) for lw in self.layers],
            embed=mv(self.embed), pos=mv(self.pos), lnf_g=mv(self.lnf_g), lnf_b=mv(self.lnf_b), meta=dict(self.meta),
        )

    def numpy_dict(self) -> dict:
        """Flat name -> fp16 ndarray map (the oracle's weight format)."""
        out = {"embed": self.embed, "pos": self.pos, "lnf.g": self.lnf_g, "lnf.b": self.lnf_b}
        for j, lw in enumerate(self.layers):
            for name, key in (("ln1.g", "ln1_g"), ("ln1.b", "ln1_b"), ("wqkv", "wqkv"), ("bqkv", "bqkv"),
                              ("wo", "wo"), ("bo", "bo"), ("ln2.g", "ln2_g"), ("ln2.b", "ln2_b"), ("w1", "w1"),
                              ("b1", "b1"), ("w2", "w2"), ("b2", "b2")):
                out[f"layers.{j}.{name}"] = getattr(lw, key)
        return {k: v.detach().cpu().numpy() for k, v in out.items()}

    def nbytes(self) -> int:
        tot = sum(t.numel() * t.element_size() for t in (self.embed, self.pos, self.lnf_g, self.lnf_b))
        for lw in self.layers:
            tot += sum(getattr(lw, k).numel() * 2 for k in lw.__dataclass_fields__)
        return tot
