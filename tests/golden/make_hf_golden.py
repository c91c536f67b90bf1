"""Pins the fp32 CPU oracle against an independent Llama implementation.

The reference (servesim) has no numeric forward, so logits cannot be pinned to
it. Instead the oracle (oracle/liboracle.so) is checked against HF transformers'
LlamaForCausalLM in fp32 (eager attention) carrying the same synthetic weights
(exported from the oracle, i.e. include/ss_synth.h). HF runs each synthetic
request's full sequence; tests/test_oracle.py replays the same tokens through
the oracle in stall-free chunks + decodes over paged KV and must reproduce
these logits.

Two shapes, each with non-unit RMSNorm gains (include/ss_synth.h):
  tiny   BASELINE configs[0]: hd 64, GQA 2, theta 1e4            -> hf_tiny_logits.npz
  hd128  the production head geometry: hd 128, GQA 4, theta 5e6
         (Yi-34B's RoPE base), sequences past 2048 positions      -> hf_hd128_gqa4_logits.npz

Run in the build container:  python tests/golden/make_hf_golden.py
Writes both .npz files (committed).
"""
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle.forward import Oracle  # noqa: E402
from paper_2403_02310_b200 import gpu, host  # noqa: E402

TOKEN_SEED = 99
WEIGHT_SEED = 1234
KEEP = 24  # logit rows kept per request (evenly spaced positions incl. the last)
# name -> (shape, sequence lengths of the three requests, output file)
CONFIGS = {
    "tiny": (gpu.MODELS["tiny"], [37, 130, 301], "hf_tiny_logits.npz"),
    "hd128": (gpu.ModelShape("hd128_gqa4", 2, 1024, 8, 2, 128, 2816, 1024, rope_theta=5e6),
              [45, 700, 2100], "hf_hd128_gqa4_logits.npz"),
}


def shape_fields(s):
    return {"shape_" + k: np.array(getattr(s, k)) for k in
            ("num_layers", "hidden", "num_q_heads", "num_kv_heads", "head_dim", "ffn", "vocab", "rope_theta",
             "rms_eps")}


def make(name):
    from transformers import LlamaConfig, LlamaForCausalLM

    s, SEQ_LENS, fname = CONFIGS[name]
    cfg = LlamaConfig(vocab_size=s.vocab, hidden_size=s.hidden, intermediate_size=s.ffn,
                      num_hidden_layers=s.num_layers, num_attention_heads=s.num_q_heads,
                      num_key_value_heads=s.num_kv_heads, head_dim=s.head_dim, max_position_embeddings=20000,
                      rms_norm_eps=s.rms_eps, rope_theta=s.rope_theta, tie_word_embeddings=False,
                      attention_bias=False, mlp_bias=False, attn_implementation="eager")
    m = LlamaForCausalLM(cfg).float().eval()
    orc = Oracle(s, weight_seed=WEIGHT_SEED, num_blocks=256)
    sd = {"model.embed_tokens.weight": orc.weight("embed"), "lm_head.weight": orc.weight("lm_head")}
    names = {"wq": "self_attn.q_proj", "wk": "self_attn.k_proj", "wv": "self_attn.v_proj", "wo": "self_attn.o_proj",
             "wg": "mlp.gate_proj", "wu": "mlp.up_proj", "wd": "mlp.down_proj"}
    for l in range(s.num_layers):
        for k, v in names.items():
            sd[f"model.layers.{l}.{v}.weight"] = orc.weight(k, l)
        sd[f"model.layers.{l}.input_layernorm.weight"] = orc.weight("attn_norm", l)[0]
        sd[f"model.layers.{l}.post_attention_layernorm.weight"] = orc.weight("mlp_norm", l)[0]
    sd["model.norm.weight"] = orc.weight("final_norm")[0]
    assert not np.allclose(sd["model.norm.weight"], 1.0)  # the gains are exercised
    missing, unexpected = m.load_state_dict({k: torch.from_numpy(v) for k, v in sd.items()}, strict=False)
    assert not unexpected and not [k for k in missing if "rotary" not in k], (missing, unexpected)

    ents = [host.BatchEntry(i, "prefill", n, 0) for i, n in enumerate(SEQ_LENS)]
    toks = host.Descriptor.build(ents, vocab=s.vocab, token_seed=TOKEN_SEED).arrays()["token_ids"]
    out = {"seq_lens": np.array(SEQ_LENS), "token_seed": TOKEN_SEED, "weight_seed": WEIGHT_SEED, **shape_fields(s)}
    off = 0
    with torch.no_grad():
        for i, n in enumerate(SEQ_LENS):
            ids = torch.from_numpy(toks[off:off + n].astype(np.int64))[None]
            logits = m(input_ids=ids).logits[0].numpy()
            # evenly spaced positions plus the last 24 (the oracle replay's decode tail)
            keep = np.unique(np.concatenate([np.linspace(0, n - 1, KEEP).round().astype(int),
                                             np.arange(max(0, n - 24), n)]))
            out[f"pos_{i}"] = keep
            out[f"logits_{i}"] = logits[keep].astype(np.float32)
            out[f"tokens_{i}"] = toks[off:off + n]
            off += n
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print("wrote", os.path.join(HERE, fname))


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CONFIGS)):
        make(n)
