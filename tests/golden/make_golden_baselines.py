"""Golden fixtures for the baseline competitors (Q/baselines.py) and the QVGC
container (Q/container.py), produced by running the REFERENCE itself.

    python tests/golden/make_golden_baselines.py

Imports the reference ``qvgcodec`` in place from /root/reference/pkg/src and
records RTN / KIVI token-axis / QuaRot payloads, scales and reconstructions,
Hadamard forward / inverse rows (float64), and the exact bytes of a QVGC
file written by the reference's ChunkWriter (QVG chunks of two configs).
The GPU box has no /root/reference, so the outputs are committed."""

from __future__ import annotations

import io
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from qvgcodec import baselines, container, prq
    from qvgcodec.lowprec import round_to_bf16
    from qvgcodec.types import ChunkSpec, KVPlane, QuantConfig

    rng = np.random.default_rng(2602)
    out = {}
    cases = [("a", 100, 128, 2, 16), ("b", 96, 128, 4, 32), ("c", 77, 64, 8, 64), ("d", 130, 128, 2, 64)]
    for name, n, d, bits, gs in cases:
        x = rng.normal(0, 2.0, size=(n, d)) * np.where(np.arange(d) % 16 == 0, 20.0, 1.0)
        x = round_to_bf16(x.astype(np.float32)).astype(np.float32)
        v = round_to_bf16(rng.normal(0, 3.0, size=(n, d)).astype(np.float32)).astype(np.float32)
        kp = KVPlane.from_array(x)
        vp = KVPlane.from_array(v)
        out[f"{name}_x"] = x
        out[f"{name}_v"] = v
        out[f"{name}_cfg"] = np.array([n, d, bits, gs])
        p, s = baselines.rtn_compress(kp, bits, gs)
        out[f"{name}_rtn_payload"] = np.frombuffer(p, np.uint8)
        out[f"{name}_rtn_scales"] = np.frombuffer(s, np.uint8)
        out[f"{name}_rtn_dec"] = baselines.rtn_decompress(p, s, n, d, bits, gs)
        kc = baselines.kivi_compress(kp, vp, bits, gs)
        out[f"{name}_kivi_kp"] = np.frombuffer(kc.keys_payload, np.uint8)
        out[f"{name}_kivi_ks"] = np.frombuffer(kc.keys_scales, np.uint8)
        out[f"{name}_kivi_vp"] = np.frombuffer(kc.values_payload, np.uint8)
        out[f"{name}_kivi_vs"] = np.frombuffer(kc.values_scales, np.uint8)
        out[f"{name}_kivi_pad"] = np.array([kc.padded_tokens])
        kk, vv = baselines.kivi_decompress(kc)
        out[f"{name}_kivi_kdec"] = kk
        out[f"{name}_kivi_vdec"] = vv
        seed = 11 + n
        qc = baselines.quarot_compress(kp, bits, gs, seed)
        out[f"{name}_quarot_payload"] = np.frombuffer(qc.payload, np.uint8)
        out[f"{name}_quarot_scales"] = np.frombuffer(qc.scales, np.uint8)
        out[f"{name}_quarot_seed"] = np.array([seed])
        out[f"{name}_quarot_dec"] = baselines.quarot_decompress(qc)
        signs = baselines.random_signs(d, seed)
        out[f"{name}_signs"] = signs
        out[f"{name}_had_fwd"] = baselines.hadamard_transform(x[:8], signs)
        out[f"{name}_had_inv"] = baselines.inverse_hadamard(x[:8], signs)
    np.savez_compressed(os.path.join(HERE, "baselines.npz"), **out)

    # QVGC container written by the reference (two QVG chunks + header)
    for tag, (cfg, n) in {"s2": (QuantConfig(bits=2, group_size=64, stages=2, centroids=8, seed=5), 64),
                          "s1b4": (QuantConfig(bits=4, group_size=32, stages=1, centroids=4), 40)}.items():
        buf = io.BytesIO()
        planes, chunks = [], []
        hdr = container.QvgcHeader.for_config(cfg, 128)
        w = container.ChunkWriter(buf, hdr)
        for c in range(2):
            x = round_to_bf16(rng.normal(0, 1.5, size=(n, 128)).astype(np.float32)).astype(np.float32)
            plane = KVPlane.from_array(x, chunk_index=c)
            ch = prq.prq_compress(plane, cfg)
            w.append_chunk(ch)
            planes.append(x)
        raw = buf.getvalue()
        np.savez_compressed(os.path.join(HERE, f"container_{tag}.npz"), qvgc=np.frombuffer(raw, np.uint8),
                            planes=np.stack(planes), cfg=np.array([cfg.bits, cfg.group_size, cfg.stages,
                                                                   cfg.centroids, cfg.seed, n]))
    print("wrote baselines.npz, container_*.npz")


if __name__ == "__main__":
    main()
