"""Synthetic fused-parameter layouts.

BERT tensors in DeepSpeed fused-QKV order, one "layer" per tensor as the
reference treats them (302 tensors for BERT-Large matches
PAPER.md:459).  Only the shapes matter: the optimizer sees a flat buffer
with a per-tensor offset table (fusion.hpp:29-44).
"""
from __future__ import annotations

VOCAB = 30522

# ragged 16-layer table, d = 8,000,003.
CONFIG1 = [2000000, 2, 1024, 1023, 1048576, 3072, 1048576, 1024, 1048576, 4096,
           1048576, 1024, 524288, 524288, 1024, 744834]


def bert_layout(hidden: int, layers: int, ffn: int, vocab: int = VOCAB) -> list[tuple[str, int]]:
    H, F = hidden, ffn
    t = [("emb.word", vocab * H), ("emb.pos", 512 * H), ("emb.type", 2 * H),
         ("emb.ln.w", H), ("emb.ln.b", H)]
    for i in range(layers):
        p = f"layer{i}."
        t += [(p + "qkv.w", 3 * H * H), (p + "qkv.b", 3 * H), (p + "attn_out.w", H * H),
              (p + "attn_out.b", H), (p + "attn_ln.w", H), (p + "attn_ln.b", H),
              (p + "inter.w", F * H), (p + "inter.b", F), (p + "out.w", H * F), (p + "out.b", H),
              (p + "out_ln.w", H), (p + "out_ln.b", H)]
    t += [("pool.w", H * H), ("pool.b", H), ("cls.transform.w", H * H), ("cls.transform.b", H),
          ("cls.ln.w", H), ("cls.ln.b", H), ("cls.bias", vocab), ("nsp.w", 2 * H), ("nsp.b", 2)]
    return t


def bert_base() -> list[tuple[str, int]]:
    return bert_layout(768, 12, 3072)


def bert_large() -> list[tuple[str, int]]:
    return bert_layout(1024, 24, 4096)


def sizes(layout) -> list[int]:
    return [s for _, s in layout]
