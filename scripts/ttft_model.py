"""TTFT projection at TP = 2/4/8 from round-1 single-GPU measurements (a
MODEL, not a measurement -- one GPU cannot run TP > 1):

    TTFT(TP) = T_body(TP=1) / TP + A * t_allreduce(TP)

T_body(TP=1): the measured CUDA-graph prefill of the random-init body with
bf16 "all-reduce" (identity at TP=1), profiles/r01/latest/ttft.jsonl;
A = 2 x layers all-reduces per prefill (o_proj, down_proj);
t_allreduce(TP): bf16 = ring wire time at 770 GB/s per direction; compressed
= the measured per-rank kernel time + modelled wire time of its bytes
(profiles/r01/latest/tp.jsonl), one-shot up to TP=2, two-shot beyond.
Perfect compute scaling and no overlap of all-reduce and compute are
assumed for both arms.
"""

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    lat = os.path.join(ROOT, "profiles", "r01", "latest")
    tp_rows = [json.loads(l) for l in open(os.path.join(lat, "tp.jsonl"))]
    ttft = [json.loads(l) for l in open(os.path.join(lat, "ttft.jsonl"))]
    body = {}
    for r in ttft:
        if r["allreduce"] == "bf16 NCCL" and r.get("cuda_graph"):
            scale = {"llama-3.1-8b": 32, "llama-3.1-70b": 80}[r["model"]] / r["layers"]
            body[r["model"]] = (r["ttft_ms"] * scale, int(r["layers"] * scale))
    shapes = {"llama-3.1-8b": [2048, 4096], "llama-3.1-70b": [4096, 8192]}
    for model, (t1, layers) in body.items():
        for tp in (2, 4, 8):
            row = next(r for r in tp_rows if r["shape"] == shapes[model] and r["tp"] == tp)
            comp = row["oneshot_us"]["total_model"] if tp <= 2 else row["twoshot_us"]["total_model"]
            bf16 = row["bf16_ring_wire_model_us"]
            a = 2 * layers
            t_bf16 = t1 / tp + a * bf16 * 1e-3
            t_comp = t1 / tp + a * comp * 1e-3
            print(json.dumps({"model": model, "tp": tp, "layers": layers,
                              "body_tp1_ms": round(t1, 2), "allreduces": a,
                              "bf16_allreduce_us": bf16, "mx_allreduce_us": comp,
                              "ttft_bf16_ms": round(t_bf16, 2), "ttft_mx_ms": round(t_comp, 2),
                              "speedup": round(t_bf16 / t_comp, 3), "kind": "model"}))


if __name__ == "__main__":
    main()
