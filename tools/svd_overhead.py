"""Fig 1c on B200 ("The relative overhead of SVD decreases as sequence length scales for the
pre-filling stage"; "the linear cost of low-rank decomposition ... negligible").

For one Llama-3.1-8B layer (32 q / 8 KV heads, d = 128, rank 160) and growing context s, times
  * shadowkv_factorize (our GPU SVD of the pre-RoPE keys: Gram on tensor cores + fp64 eigensolve +
    projection), and
  * the layer's causal prefill attention (torch SDPA, a library kernel used only as the yardstick),
with CUDA events (median of 5 after a warm-up) and prints one JSON line per length plus a summary.

  python tools/svd_overhead.py [--lengths 8192,16384,...]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_21465_b200 import LayerState, RopeTable, Shape, alloc_workspace, factorize  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="8192,16384,32768,65536,131072,262144")
    ap.add_argument("--rank", type=int, default=160)
    args = ap.parse_args()
    hq, hk, d = 32, 8, 128
    rows = []
    for s in [int(x) for x in args.lengths.split(",")]:
        g = torch.Generator(device="cuda").manual_seed(s)
        K = torch.randn(1, hk, s, d, device="cuda", generator=g, dtype=torch.float32).to(torch.bfloat16)
        t_svd = timed(lambda: factorize(K, args.rank))
        # the rest of Alg 1 on the factors: landmarks, min-cos, outliers, window (shadowkv_build_cache)
        A, B, _ = factorize(K, args.rank)
        cfg = synth.CONFIGS["c2"].replace(ctx_len=s, budget=max(1, s // 512))
        shape = Shape.from_config(cfg, steps=1)
        st = LayerState(shape)
        st.A.copy_(A); st.B.copy_(B)
        inv, rot, il = synth.rope_table(cfg)
        rope = RopeTable(inv, rot, il)
        ws = alloc_workspace(shape)
        t_build = timed(lambda: st.build(rope.struct, ws))
        del st, ws, A, B
        q = torch.randn(1, hq, s, d, device="cuda", generator=g, dtype=torch.float32).to(torch.bfloat16)
        v = torch.randn(1, hk, s, d, device="cuda", generator=g, dtype=torch.float32).to(torch.bfloat16)
        attn = lambda: torch.nn.functional.scaled_dot_product_attention(q, K, v, is_causal=True, enable_gqa=True)
        t_att = timed(attn, reps=3)
        flops = 4.0 * hq * d * s * s / 2                    # causal
        row = {"ctx": s, "svd_ms": t_svd, "build_ms": t_build, "prefill_attn_ms": t_att,
               "svd_over_attn": t_svd / t_att, "svd_plus_build_over_attn": (t_svd + t_build) / t_att,
               "attn_tflops": flops / (t_att * 1e-3) / 1e12,
               "gram_tflops": 2.0 * s * (hk * d) ** 2 / (t_svd * 1e-3) / 1e12}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del K, q, v
        torch.cuda.empty_cache()
    print(json.dumps({"summary": "(svd + build) / attention time ratio by context",
                      "ratios": {r["ctx"]: round(r["svd_plus_build_over_attn"], 4) for r in rows}}))


if __name__ == "__main__":
    main()
