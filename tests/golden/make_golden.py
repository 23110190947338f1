"""Generate golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference ``qvgcodec`` package in place from
/root/reference/pkg/src (pure Python + numpy) and records, for a set of
seeded planes, every value the hot path produces: k-means++ picks,
per-stage iteration counts / objectives / f64 centroids (through the
reference's own ``kmeans``), the ``prq_compress`` chunk (payload, scales,
bf16 centroids, assignments) and ``prq_decompress_onepass`` output, plus
FP8 / quantizer known answers.  The GPU box has no /root/reference, so the
fixtures (``*.npz``) are committed next to this script.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import qvgcodec  # noqa: F401
    from qvgcodec import clustering, datagen, lowprec, prq, quant, types

    return clustering, datagen, lowprec, prq, quant, types


def plane_cases(datagen, lowprec):
    """(name, data f32 (N,d) bf16-exact, cfg dict, chunk_index, warm_from)"""
    cases = []

    def clustered(n, d, nclu, scale, seed, chunks=1, drift=0.0):
        planes = datagen.gen_clustered_stream(
            n_chunks=chunks, n_tokens=n, d=d, n_clusters=nclu, sigma_within=0.125,
            sigma_between=2.5, drift=drift, outlier_channels=tuple(range(0, d, 16)),
            outlier_scale=scale, seed=seed)
        return [lowprec.round_to_bf16(p.data) for p in planes]

    # C1-shaped planes (config 1: N 4680, K 64, S 2, b 2, B 64), one K and one V plane
    c1 = dict(bits=2, group_size=64, stages=2, centroids=64)
    cases.append(("c1_key", clustered(4680, 128, 256, 10.0, 0)[0], c1, 0))
    cases.append(("c1_value", clustered(4680, 128, 256, 100.0, 1)[0], c1, 0))
    # smaller shapes across the knob space
    cases.append(("s2_b4_g16", clustered(1000, 64, 40, 10.0, 2)[0],
                  dict(bits=4, group_size=16, stages=1, centroids=32), 3))
    cases.append(("s3_b8_g32", clustered(600, 128, 20, 100.0, 3)[0],
                  dict(bits=8, group_size=32, stages=3, centroids=8), 1))
    cases.append(("s4_pro", clustered(512, 128, 64, 100.0, 4)[0],
                  dict(bits=2, group_size=16, stages=4, centroids=16), 2))
    cases.append(("k256", clustered(2048, 128, 256, 100.0, 5)[0],
                  dict(bits=2, group_size=64, stages=1, centroids=256), 0))
    cases.append(("k1", clustered(300, 32, 5, 1.0, 6)[0],
                  dict(bits=4, group_size=32, stages=2, centroids=1), 0))
    cases.append(("s0_rtn_saturate", clustered(256, 128, 16, 100.0, 7)[0],
                  dict(bits=2, group_size=64, stages=0, centroids=4), 0))
    # edge cases: fewer rows than centroids (uniform fallback + empty repair),
    # duplicated rows (exact distance ties), zero plane, one row, odd d
    rng = np.random.default_rng(8)
    cases.append(("n_lt_k", lowprec.round_to_bf16(rng.normal(size=(10, 16)).astype(np.float32)),
                  dict(bits=2, group_size=16, stages=1, centroids=16), 0))
    base = rng.normal(scale=3.0, size=(4, 128)).astype(np.float32)
    dup = lowprec.round_to_bf16(np.repeat(base, 16, axis=0)[rng.permutation(64)])
    cases.append(("ties", dup, dict(bits=2, group_size=64, stages=2, centroids=8), 0))
    cases.append(("zero", np.zeros((64, 32), np.float32),
                  dict(bits=2, group_size=16, stages=1, centroids=4), 0))
    cases.append(("one_row", lowprec.round_to_bf16(rng.normal(size=(1, 128)).astype(np.float32)),
                  dict(bits=2, group_size=64, stages=1, centroids=1), 0))
    cases.append(("d24", lowprec.round_to_bf16((rng.normal(size=(333, 24)) * 4).astype(np.float32)),
                  dict(bits=4, group_size=8, stages=2, centroids=5), 4))
    # streaming pair for warm start: chunk 1 warm-started from chunk 0's f64 centroids
    stream = clustered(1024, 128, 32, 10.0, 9, chunks=2, drift=0.0125)
    cases.append(("warm0", stream[0], dict(bits=2, group_size=64, stages=2, centroids=32), 0))
    cases.append(("warm1", stream[1], dict(bits=2, group_size=64, stages=2, centroids=32), 1))
    return cases


def main():
    clustering, datagen, lowprec, prq, quant, types = _ref()
    out = {}

    # --- FP8 / bf16 / quantizer known answers -------------------------------
    rng = np.random.default_rng(100)
    mags = np.concatenate([10.0 ** rng.uniform(-12, 4, size=4000),
                           [lowprec.fp8_e4m3_decode(c) for c in range(0x7F)],
                           [1 / 7, 1e-9, 2.0 ** -10, 448.0, 448.5, 1000.0, 0.0]])
    out["fp8_x"] = mags
    out["fp8_up"] = lowprec.fp8_e4m3_encode_array(mags, "up")
    out["fp8_nearest"] = lowprec.fp8_e4m3_encode_array(mags, "nearest")
    f = (rng.normal(size=5000) * 10.0 ** rng.uniform(-30, 30, size=5000)).astype(np.float32)
    out["bf16_in"] = f
    out["bf16_out"] = lowprec.round_to_bf16(f)
    for bits in (2, 4, 8):
        for g in (8, 16, 64, 128):
            x = rng.normal(size=(37, 128)) * 10.0 ** rng.uniform(-3, 3, size=(37, 1))
            x[3] = 0.0
            x[5, :g] = 0.0
            p, s = quant.quantize_matrix(x, types.QuantConfig(bits=bits, group_size=g))
            out[f"qm_b{bits}_g{g}_x"] = x
            out[f"qm_b{bits}_g{g}_payload"] = np.frombuffer(p, np.uint8)
            out[f"qm_b{bits}_g{g}_scales"] = np.frombuffer(s, np.uint8)
            out[f"qm_b{bits}_g{g}_deq"] = quant.dequantize_plane(p, s, 37, 128, bits, g)
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)

    # --- per-plane PRQ trajectories ----------------------------------------
    names = []
    for name, data, cfgd, chunk in plane_cases(datagen, lowprec):
        cfg = types.QuantConfig(**cfgd)
        plane = types.KVPlane.from_array(data, chunk_index=chunk)
        warm = None
        assert np.array_equal(lowprec.round_to_bf16(data), data)
        rec = {"x_bf16": lowprec.bf16_pack(data), "chunk_index": chunk}
        for key, val in cfgd.items():
            rec["cfg_" + key] = val
        if name == "warm1":
            prev = np.load(os.path.join(HERE, "plane_warm0.npz"))
            warm = [prev["cent_f64"][t] for t in range(cfg.stages)]
            rec["warm"] = np.stack(warm)
        chunk_obj = prq.prq_compress(plane, cfg, warm_init=warm)
        rec["payload"] = np.frombuffer(chunk_obj.payload, np.uint8)
        rec["scales"] = np.frombuffer(chunk_obj.scales, np.uint8)
        d = data.shape[1]
        rec["centroids"] = (np.stack([m.centroids for m in chunk_obj.stages])
                            if cfg.stages else np.zeros((0, cfg.centroids, d), np.float32))
        rec["assignments"] = (np.stack([m.assignments for m in chunk_obj.stages])
                              if cfg.stages else np.zeros((0, data.shape[0]), np.uint8))
        rec["decoded"] = prq.prq_decompress_onepass(chunk_obj).data
        # replay the chain through the reference internals to record the trajectory
        resid = data.astype(np.float64)
        picks, iters, objs, c64 = [], [], [], []
        for t in range(1, cfg.stages + 1):
            seed = prq.stage_seed(cfg.seed, chunk, t)
            if warm is None:
                init = clustering.kmeans_pp_init(resid, cfg.centroids, seed)
                chosen = [int(np.flatnonzero((resid == r).all(axis=1))[0]) for r in init]
                picks.append(chosen)
            res = clustering.kmeans(resid, cfg.centroids, cfg.kmeans_max_iters, cfg.kmeans_tol,
                                    seed=seed, init=None if warm is None else warm[t - 1])
            iters.append(res.iterations_used)
            objs.append(res.objective)
            c64.append(res.centroids)
            cb = lowprec.round_to_bf16(res.centroids.astype(np.float32))
            assert np.array_equal(cb, rec["centroids"][t - 1])
            resid = resid - cb[res.assignments].astype(np.float64)
        rec["iters"] = np.array(iters, np.int32)
        rec["objective"] = np.array(objs, np.float64)
        rec["cent_f64"] = (np.stack(c64) if c64 else np.zeros((0, cfg.centroids, d)))
        if picks:
            rec["pp_first_picks"] = np.array(picks, np.int64)
        np.savez_compressed(os.path.join(HERE, f"plane_{name}.npz"), **rec)
        names.append(name)
        print(name, data.shape, cfgd, "iters", iters, flush=True)
    with open(os.path.join(HERE, "MANIFEST.txt"), "w") as fh:
        fh.write("# fixtures written by make_golden.py from the reference at " + REF + "\n")
        for n in names:
            fh.write(f"plane_{n}.npz\n")
        fh.write("kat.npz\n")


if __name__ == "__main__":
    main()
