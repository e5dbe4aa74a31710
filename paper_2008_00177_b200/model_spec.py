"""BERT parameter-set shapes for the synthetic gradient-to-update workload.

Restates the parameter list of the reference's ``build_model``
(proj/core/src/model.cpp:124-176): names, shapes, order and init kind, and the
order in which the forward pass first consumes each parameter
(proj/core/src/model.cpp:257-325 with amp=false). The first-use order is what
``BucketLayout::build`` (trainer.cpp:73-116) sorts on: gradients become final
in reverse first-use order.

Only shapes matter to the hot path; no forward pass is built here.
"""
from __future__ import annotations

from dataclasses import dataclass, field

RANDN, ONES, ZEROS = 0, 1, 2


@dataclass(frozen=True)
class ModelConfig:
    """Mirror of ``bertopt::ModelConfig`` (model.hpp:33-44)."""

    layers: int = 2
    hidden: int = 64
    heads: int = 4
    vocab: int = 1000
    max_seq: int = 512

    def intermediate(self) -> int:
        return 4 * self.hidden


BERT_LARGE = ModelConfig(layers=24, hidden=1024, heads=16, vocab=30522, max_seq=512)
BERT_LARGE_PHASE1 = ModelConfig(layers=24, hidden=1024, heads=16, vocab=30522, max_seq=128)
BERT_BASE = ModelConfig(layers=12, hidden=768, heads=12, vocab=30522, max_seq=512)
BERT_TINY = ModelConfig(layers=2, hidden=64, heads=4, vocab=1000, max_seq=64)


@dataclass
class ModelSpec:
    names: list[str] = field(default_factory=list)
    shapes: list[tuple[int, ...]] = field(default_factory=list)
    init: list[int] = field(default_factory=list)
    first_use: list[int] = field(default_factory=list)  # tensor ids, forward first-use order

    @property
    def n_tensors(self) -> int:
        return len(self.names)

    def numels(self) -> list[int]:
        out = []
        for s in self.shapes:
            n = 1
            for d in s:
                n *= d
            out.append(n)
        return out

    def param_count(self) -> int:
        return sum(self.numels())

    def first_consumer_ids(self) -> list[int]:
        """A first-consumer op id per tensor (the rank in first-use order)."""
        ids = [0] * self.n_tensors
        for pos, t in enumerate(self.first_use):
            ids[t] = pos
        return ids

    def index(self, name: str) -> int:
        return self.names.index(name)


def bert_spec(cfg: ModelConfig) -> ModelSpec:
    d, di, V = cfg.hidden, cfg.intermediate(), cfg.vocab
    spec = ModelSpec()

    def add(name: str, shape: tuple[int, ...], init: int) -> None:
        spec.names.append(name)
        spec.shapes.append(shape)
        spec.init.append(init)

    # build_model order (model.cpp:140-174).
    add("embedding.word", (V, d), RANDN)
    add("embedding.position", (cfg.max_seq, d), RANDN)
    add("embedding.segment", (2, d), RANDN)
    add("embedding.ln_gamma", (d,), ONES)
    add("embedding.ln_beta", (d,), ZEROS)
    for layer in range(cfg.layers):
        p = f"layer{layer}"
        for w in ("q", "k", "v", "o"):
            add(f"{p}.attention.w{w}", (d, d), RANDN)
            add(f"{p}.attention.b{w}", (d,), ZEROS)
        add(f"{p}.attention.ln_gamma", (d,), ONES)
        add(f"{p}.attention.ln_beta", (d,), ZEROS)
        add(f"{p}.intermediate.w", (d, di), RANDN)
        add(f"{p}.intermediate.b", (di,), ZEROS)
        add(f"{p}.output.w", (di, d), RANDN)
        add(f"{p}.output.b", (d,), ZEROS)
        add(f"{p}.output.ln_gamma", (d,), ONES)
        add(f"{p}.output.ln_beta", (d,), ZEROS)
    add("mlm.transform_w", (d, d), RANDN)
    add("mlm.transform_b", (d,), ZEROS)
    add("mlm.ln_gamma", (d,), ONES)
    add("mlm.ln_beta", (d,), ZEROS)
    add("mlm.bias", (V,), ZEROS)
    add("pooler.w", (d, d), RANDN)
    add("pooler.b", (d,), ZEROS)
    add("nsp.w", (d, 2), RANDN)
    add("nsp.b", (2,), ZEROS)

    # Forward first-use order (model.cpp:257-325, amp=false): embeddings,
    # then per layer q,k,v projections (w before b), output projection, the
    # attention LN (gamma, beta), FFN, output LN; pooler and NSP head before
    # the MLM head, whose decoder reuses embedding.word and adds mlm.bias last.
    order = ["embedding.word", "embedding.position", "embedding.segment",
             "embedding.ln_gamma", "embedding.ln_beta"]
    for layer in range(cfg.layers):
        p = f"layer{layer}"
        order += [f"{p}.attention.wq", f"{p}.attention.bq", f"{p}.attention.wk",
                  f"{p}.attention.bk", f"{p}.attention.wv", f"{p}.attention.bv",
                  f"{p}.attention.wo", f"{p}.attention.bo", f"{p}.attention.ln_gamma",
                  f"{p}.attention.ln_beta", f"{p}.intermediate.w", f"{p}.intermediate.b",
                  f"{p}.output.w", f"{p}.output.b", f"{p}.output.ln_gamma",
                  f"{p}.output.ln_beta"]
    order += ["pooler.w", "pooler.b", "nsp.w", "nsp.b", "mlm.transform_w",
              "mlm.transform_b", "mlm.ln_gamma", "mlm.ln_beta", "mlm.bias"]
    pos = {n: i for i, n in enumerate(spec.names)}
    spec.first_use = [pos[n] for n in order]
    assert sorted(spec.first_use) == list(range(spec.n_tensors))
    return spec


def flat_spec(numels: list[int], first_use: list[int] | None = None) -> ModelSpec:
    """A spec of 1-D tensors with the given sizes (for edge-case tests)."""
    spec = ModelSpec()
    for i, n in enumerate(numels):
        spec.names.append(f"t{i}")
        spec.shapes.append((n,))
        spec.init.append(RANDN)
    spec.first_use = list(first_use) if first_use is not None else list(range(len(numels)))
    return spec
