"""Pins the fp32 CPU oracle against an independent Llama implementation.

The reference (servesim) has no numeric forward, so logits cannot be pinned to
it. Instead the oracle (oracle/liboracle.so) is checked against HF transformers'
LlamaForCausalLM in fp32 (eager attention) carrying the same synthetic weights
(exported from the oracle, i.e. include/ss_synth.h). HF runs each synthetic
request's full sequence; tests/test_oracle.py replays the same tokens through
the oracle in stall-free chunks + decodes over paged KV and must reproduce
these logits.

Run in the build container:  python tests/golden/make_hf_golden.py
Writes tests/golden/hf_tiny_logits.npz (committed).
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

SEQ_LENS = [37, 130, 301]  # three requests, token ids ss_token_id(seed, rid, pos)
TOKEN_SEED = 99
WEIGHT_SEED = 1234
KEEP = 24  # logit rows kept per request (evenly spaced positions incl. the last)


def main():
    from transformers import LlamaConfig, LlamaForCausalLM

    s = gpu.MODELS["tiny"]
    cfg = LlamaConfig(vocab_size=s.vocab, hidden_size=s.hidden, intermediate_size=s.ffn,
                      num_hidden_layers=s.num_layers, num_attention_heads=s.num_q_heads,
                      num_key_value_heads=s.num_kv_heads, head_dim=s.head_dim, max_position_embeddings=20000,
                      rms_norm_eps=s.rms_eps, rope_theta=s.rope_theta, tie_word_embeddings=False,
                      attention_bias=False, mlp_bias=False, attn_implementation="eager")
    m = LlamaForCausalLM(cfg).float().eval()
    orc = Oracle(s, weight_seed=WEIGHT_SEED, num_blocks=64)
    sd = {"model.embed_tokens.weight": orc.weight("embed"), "lm_head.weight": orc.weight("lm_head")}
    names = {"wq": "self_attn.q_proj", "wk": "self_attn.k_proj", "wv": "self_attn.v_proj", "wo": "self_attn.o_proj",
             "wg": "mlp.gate_proj", "wu": "mlp.up_proj", "wd": "mlp.down_proj"}
    for l in range(s.num_layers):
        for k, v in names.items():
            sd[f"model.layers.{l}.{v}.weight"] = orc.weight(k, l)
        sd[f"model.layers.{l}.input_layernorm.weight"] = np.ones(s.hidden, np.float32)
        sd[f"model.layers.{l}.post_attention_layernorm.weight"] = np.ones(s.hidden, np.float32)
    sd["model.norm.weight"] = np.ones(s.hidden, np.float32)
    missing, unexpected = m.load_state_dict({k: torch.from_numpy(v) for k, v in sd.items()}, strict=False)
    assert not unexpected and not [k for k in missing if "rotary" not in k], (missing, unexpected)

    ents = [host.BatchEntry(i, "prefill", n, 0) for i, n in enumerate(SEQ_LENS)]
    toks = host.Descriptor.build(ents, vocab=s.vocab, token_seed=TOKEN_SEED).arrays()["token_ids"]
    out = {"seq_lens": np.array(SEQ_LENS), "token_seed": TOKEN_SEED, "weight_seed": WEIGHT_SEED}
    off = 0
    with torch.no_grad():
        for i, n in enumerate(SEQ_LENS):
            ids = torch.from_numpy(toks[off:off + n].astype(np.int64))[None]
            logits = m(input_ids=ids).logits[0].numpy()
            keep = np.unique(np.linspace(0, n - 1, KEEP).round().astype(int))
            out[f"pos_{i}"] = keep
            out[f"logits_{i}"] = logits[keep].astype(np.float32)
            out[f"tokens_{i}"] = toks[off:off + n]
            off += n
    np.savez_compressed(os.path.join(HERE, "hf_tiny_logits.npz"), **out)
    print("wrote", os.path.join(HERE, "hf_tiny_logits.npz"))


if __name__ == "__main__":
    main()
