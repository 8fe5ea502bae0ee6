"""Generate the golden fixtures from the REAL reference (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [/root/reference/pkg/src]

Imports the unmodified reference package ``embquant`` read-only and records
its outputs for the hot path (ASYM / GREEDY / HIST-BRUTE clip ranges, the
uniform codec, pack_table4 bytes, WorkCounters, quant_mse values) on seeded
inputs.  The fixtures are committed; /root/reference does not exist on the GPU
box, so tests there compare against these files and against the C oracle that
these files pin.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import embquant as eq  # noqa: E402
from embquant.rng import derive_seed, uniform_open01  # noqa: E402
from embquant.uniform import quantize_table_uniform  # noqa: E402

sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.rng import mixed_table  # noqa: E402  (plain numpy Generator recipe)


def gaussian_rows(seed, rows, d, scale=1.0, loc=0.0):
    return eq.sample_table(eq.RngSpec("gaussian", loc, scale, seed), rows, d).values.copy()


def laplacian_rows(seed, rows, d, scale=1.0):
    return eq.sample_table(eq.RngSpec("laplacian", 0.0, scale, seed), rows, d).values.copy()


def ref_greedy(x, b, r, aux):
    """pack_table4(quantize_table(t, 'greedy', 4, aux, b, r)) + per-row ranges/counters."""
    t = eq.EmbeddingTable(x)
    lo, hi, ev = [], [], []
    for i in range(t.rows):
        c = eq.WorkCounters()
        cr = eq.clip_range_greedy(t.row(i), 4, b, r, counters=c)
        lo.append(cr.xmin)
        hi.append(cr.xmax)
        ev.append(c.loss_evals)
    q = eq.quantize_table(t, "greedy", 4, aux, b, r)
    return eq.pack_table4(q).buffer.copy(), np.array(lo), np.array(hi), np.array(ev, np.int64)


def ref_asym(x, aux):
    t = eq.EmbeddingTable(x)
    q = eq.quantize_table(t, "asym", 4, aux)
    lo = np.array([eq.clip_range_asym(t.row(i)).xmin for i in range(t.rows)])
    hi = np.array([eq.clip_range_asym(t.row(i)).xmax for i in range(t.rows)])
    return eq.pack_table4(q).buffer.copy(), lo, hi


def ref_hist(x, b, aux="fp16"):
    t = eq.EmbeddingTable(x)
    out = {k: [] for k in ("lo", "hi", "start", "n", "norm", "cand", "visits")}
    for i in range(t.rows):
        c = eq.WorkCounters()
        w = eq.hist_brute_search(t.row(i), b, counters=c)
        out["lo"].append(w.clip_range.xmin)
        out["hi"].append(w.clip_range.xmax)
        out["start"].append(w.start_bin)
        out["n"].append(w.nbins_selected)
        out["norm"].append(w.norm)
        out["cand"].append(c.candidate_evals)
        out["visits"].append(c.bin_visits)
    ranges = [eq.ClipRange(a, b_) for a, b_ in zip(out["lo"], out["hi"])]
    packed = eq.pack_table4(quantize_table_uniform(t, ranges, 4, aux, "hist-brute")).buffer.copy()
    res = {k: np.array(v) for k, v in out.items()}
    res["packed"] = packed
    return res


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_config1():
    t0 = time.time()
    x = gaussian_rows(1911, 10000, 64)
    out = {"table_sha256": np.array(sha(x)), "head": x[:16].copy()}
    out["greedy_fp16_packed"], out["greedy_lo"], out["greedy_hi"], out["greedy_evals"] = \
        ref_greedy(x, 200, 0.16, "fp16")
    t = eq.EmbeddingTable(x)
    ranges = [eq.ClipRange(a, b) for a, b in zip(out["greedy_lo"], out["greedy_hi"])]
    out["greedy_fp32_packed"] = eq.pack_table4(quantize_table_uniform(t, ranges, 4, "fp32")).buffer
    out["asym_fp16_packed"], _, _ = ref_asym(x, "fp16")
    out["asym_fp32_packed"], _, _ = ref_asym(x, "fp32")
    # laplacian port pin
    lap = laplacian_rows(77, 64, 64)
    out["laplacian_sha256"] = np.array(sha(lap))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)
    print(f"config1: {time.time() - t0:.1f}s")


def edge_inputs():
    """(name, x, b, r) greedy/asym edge cases; x is (rows, d) float32."""
    cases = []
    cases.append(("exact_grid", np.arange(16, dtype=np.float32)[None], 200, 0.16))
    g = gaussian_rows(13, 1, 63)[0]
    cases.append(("outlier", np.concatenate([g, np.float32([100.0])])[None], 200, 0.16))
    cases.append(("constant", np.array([[4.0, 4.0], [2.5, 2.5]], np.float32), 200, 0.16))
    cases.append(("constant_wide", np.full((2, 37), -1.25, np.float32), 200, 0.16))
    for i, d in enumerate([1, 2, 3, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 48, 63, 64, 65, 100, 127,
                           128, 129, 200, 255, 256, 257, 300, 511, 512, 1000, 1024, 2048]):
        rows = 6 if d <= 512 else 3
        cases.append((f"gauss_d{d}", gaussian_rows(derive_seed(5, d), rows, d), 200, 0.16))
    cases.append(("laplacian_d64", laplacian_rows(91, 64, 64), 200, 0.16))
    cases.append(("offset_1000", (1000.0 + gaussian_rows(17, 16, 64) * 1e-3).astype(np.float32),
                  200, 0.16))
    cases.append(("tiny_1e-30", (gaussian_rows(18, 8, 32) * 1e-30).astype(np.float32), 200, 0.16))
    cases.append(("subnormal", (gaussian_rows(19, 4, 16) * 1e-41).astype(np.float32), 200, 0.16))
    cases.append(("huge_1e30", (gaussian_rows(20, 8, 32) * 1e30).astype(np.float32), 200, 0.16))
    u = uniform_open01(21, 16 * 64).reshape(16, 64)
    cases.append(("half_grid", (np.floor(u * 31) / 2).astype(np.float32), 200, 0.16))
    cases.append(("few_values", (np.floor(u * 5) - 2).astype(np.float32), 200, 0.16))
    gs = gaussian_rows(22, 8, 32)
    cases.append(("symmetric", np.concatenate([gs, -gs], 1), 200, 0.16))
    cases.append(("mixed_d128", mixed_table(384, 128, 1911), 200, 0.16))
    cases.append(("mixed_d64", mixed_table(384, 64, 1912), 200, 0.16))
    base = gaussian_rows(23, 12, 64)
    odd = gaussian_rows(24, 6, 17)
    for b, r in [(1, 0.16), (1, 1.0), (2, 1.0), (3, 0.9), (8, 0.5), (16, 0.16), (40, 0.16),
                 (64, 0.16), (200, 0.01), (200, 0.5), (200, 1.0), (400, 0.16), (1000, 0.5)]:
        cases.append((f"b{b}_r{r}", base, b, r))
        cases.append((f"b{b}_r{r}_d17", odd, b, r))
    return cases


def make_edge():
    t0 = time.time()
    out = {}
    meta = []
    for k, (name, x, b, r) in enumerate(edge_inputs()):
        x = np.ascontiguousarray(x, np.float32)
        out[f"x_{k}"] = x
        m = {"name": name, "b": b, "r": r, "greedy_error": None}
        for aux in ("fp16", "fp32"):
            try:
                p, lo, hi, ev = ref_greedy(x, b, r, aux)
                out[f"greedy_{aux}_{k}"] = p
                out[f"greedy_lo_{k}"], out[f"greedy_hi_{k}"], out[f"greedy_evals_{k}"] = lo, hi, ev
            except ValueError as e:
                m["greedy_error"] = str(e)
            p, lo, hi = ref_asym(x, aux)
            out[f"asym_{aux}_{k}"] = p
        meta.append(m)
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "edge.npz"), **out)
    print(f"edge: {len(meta)} cases {time.time() - t0:.1f}s")


def make_hist():
    t0 = time.time()
    cases = []
    for b in (8, 16, 40):
        cases.append((f"gauss_b{b}", np.stack([gaussian_rows(s * 31 + 1, 1, 64)[0] for s in range(5)]), b))
    cases.append(("lap_b16_d100", laplacian_rows(5, 6, 100), 16))
    cases.append(("gauss_b64_d32", gaussian_rows(6, 6, 32), 64))
    cases.append(("gauss_b200_d17", gaussian_rows(7, 4, 17), 200))
    dense = uniform_open01(123, 4000).astype(np.float32)
    cases.append(("outlier_prefix_b40", np.concatenate([dense, np.float32([25.0])])[None], 40))
    cases.append(("constant_b16", np.full((1, 3), 4.0, np.float32), 16))
    cases.append(("exact_grid_b16", np.arange(16, dtype=np.float32)[None], 16))
    cases.append(("b1", gaussian_rows(8, 3, 64), 1))
    cases.append(("config4_b200", gaussian_rows(2024, 256, 64), 200))
    out = {}
    meta = []
    for k, (name, x, b) in enumerate(cases):
        x = np.ascontiguousarray(x, np.float32)
        out[f"x_{k}"] = x
        res = ref_hist(x, b)
        for key, v in res.items():
            out[f"{key}_{k}"] = v
        meta.append({"name": name, "b": b})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "hist.npz"), **out)
    print(f"hist: {time.time() - t0:.1f}s")


def make_mse():
    """quant_mse values (table.py:81-103) for random rows/ranges: pins the f64 op order + np.sum."""
    rng = np.random.default_rng(7)
    xs, lo, hi, nb, val, dims = [], [], [], [], [], []
    for i in range(1500):
        d = int(rng.integers(1, 300)) if i % 5 else int(rng.choice([64, 128, 129, 256, 1000, 2048]))
        x = (rng.standard_normal(d) * 10.0 ** rng.uniform(-3, 3)).astype(np.float32)
        a, b = float(x.min()), float(x.max())
        if i % 7 == 0:
            l, h = a, a
        else:
            w = b - a
            l = a + w * rng.uniform(0, 0.3)
            h = b - w * rng.uniform(0, 0.3)
            if l > h:
                l, h = h, l
        n = 8 if i % 11 == 0 else 4
        xs.append(x); lo.append(l); hi.append(h); nb.append(n); dims.append(d)
        val.append(eq.quant_mse(x, eq.ClipRange(l, h), n))
    out = {"x": np.concatenate(xs), "dims": np.array(dims), "lo": np.array(lo), "hi": np.array(hi),
           "nbits": np.array(nb), "value": np.array(val)}
    np.savez_compressed(os.path.join(HERE, "quant_mse.npz"), **out)
    print("quant_mse: done")


def make_sls():
    """sparse_lengths_sum_4bit over packed tables (packed.py:167-177), checked against
    sparse_lengths_sum_ref (packed.py:202-221), plus the reference's error texts."""
    from embquant.packed import PooledQuery, sparse_lengths_sum_4bit, sparse_lengths_sum_ref
    from embquant.uniform import UniformQuantTable

    rng = np.random.default_rng(11)
    bufs, outs, idxs, lens, meta = [], [], [], [], []
    for case in range(400):
        rows = int(rng.integers(1, 7)) if case % 4 else int(rng.integers(7, 60))
        d = int(rng.integers(1, 41)) if case % 10 else int(rng.choice([64, 96, 128, 256, 2048]))
        aux = "fp32" if case % 3 else "fp16"
        codes = rng.integers(0, 16, size=(rows, d)).astype(np.uint8)
        scales = 0.01 + rng.integers(0, 1000, size=rows) / 250.0 * 10.0 ** rng.uniform(-3, 2)
        biases = -2.0 + rng.integers(0, 1000, size=rows) / 250.0 * 10.0 ** rng.uniform(-3, 2)
        q = UniformQuantTable(codes, scales, biases, 4, aux)
        packed = eq.pack_table4(q)
        batch = int(rng.integers(1, 6))
        ln = rng.integers(0, 5, size=batch)
        if case % 17 == 0:
            ln[:] = 0
        idx = rng.integers(0, rows, size=int(ln.sum()))
        query = PooledQuery(idx, ln)
        got = sparse_lengths_sum_4bit(packed, query)
        want = sparse_lengths_sum_ref(packed, query)
        assert np.array_equal(got, want)
        bufs.append(packed.buffer.copy()); outs.append(got.ravel()); idxs.append(idx); lens.append(ln)
        meta.append((rows, d, 1 if aux == "fp16" else 0, batch, idx.size))
    errs = {}
    packed = eq.pack_table4(UniformQuantTable(np.zeros((4, 6), np.uint8), np.ones(4), np.zeros(4), 4, "fp16"))
    for name, (i, l) in {"oob": ([0, 1, 9], [3]), "neg": ([0, 1], [-1, 2])}.items():
        try:
            sparse_lengths_sum_4bit(packed, PooledQuery(i, l))
        except (IndexError, ValueError) as e:
            errs[name] = f"{type(e).__name__}: {e}"
    try:
        PooledQuery([1, 2], [1])
    except ValueError as e:
        errs["sum"] = f"ValueError: {e}"
    out = {"packed": np.concatenate(bufs), "out": np.concatenate(outs), "indices": np.concatenate(idxs),
           "lengths": np.concatenate(lens), "meta": np.array(meta, np.int64),
           "errors": np.array(json.dumps(errs))}
    np.savez_compressed(os.path.join(HERE, "sls.npz"), **out)
    print("sls: done", errs)


def make_files():
    """EMBT / EMBQ container bytes and DataError texts (fileio.py) from the reference."""
    import tempfile

    from embquant import fileio

    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        def path(name):
            return os.path.join(tmp, name)

        x = gaussian_rows(4242, 37, 9)
        t = eq.EmbeddingTable(x)
        fileio.write_embt(path("t.embt"), t)
        out["embt"] = np.frombuffer(open(path("t.embt"), "rb").read(), np.uint8)
        for name, method, aux in (("greedy_fp16", "greedy", "fp16"), ("asym_fp32", "asym", "fp32"),
                                  ("hist_fp16", "hist-brute", "fp16")):
            q = eq.quantize_table(t, method, 4, aux)
            fileio.write_embq(path(name), q)
            out["embq_" + name] = np.frombuffer(open(path(name), "rb").read(), np.uint8)
        good = bytes(out["embt"])
        cases = {
            "embt_short": good[:20],
            "embt_magic": b"EMBX" + good[4:],
            "embt_version": good[:4] + (2).to_bytes(4, "little") + good[8:],
            "embt_dtype": good[:24] + b"\x01" + good[25:],
            "embt_shape": good[:8] + (0).to_bytes(8, "little") + good[16:],
            "embt_payload": good[:-4],
            "embt_nonfinite": good[:25] + np.array([np.nan], "<f4").tobytes() + good[29:],
        }
        msgs = {}
        for k, blob in cases.items():
            with open(path(k), "wb") as fh:
                fh.write(blob)
            try:
                fileio.read_embt(path(k))
            except fileio.DataError as e:
                msgs[k] = str(e).replace(tmp, "<dir>")
            out["bad_" + k] = np.frombuffer(blob, np.uint8)
        gq = bytes(out["embq_greedy_fp16"])
        qcases = {
            "embq_short": gq[:10],
            "embq_magic": b"EMBT" + gq[4:],
            "embq_version": gq[:4] + (9).to_bytes(4, "little") + gq[8:],
            "embq_scheme": gq[:8] + b"\x07" + gq[9:],
            "embq_aux": gq[:9] + b"\x05" + gq[10:],
            "embq_shape": gq[:18] + (0).to_bytes(8, "little") + gq[26:],
            "embq_truncated": gq[:-1],
            "embq_mismatch": gq + b"\x00",
        }
        for k, blob in qcases.items():
            with open(path(k), "wb") as fh:
                fh.write(blob)
            try:
                fileio.read_embq(path(k))
            except fileio.DataError as e:
                msgs[k] = str(e).replace(tmp, "<dir>")
            out["bad_" + k] = np.frombuffer(blob, np.uint8)
    out["table"] = x
    out["messages"] = np.array(json.dumps(msgs))
    np.savez_compressed(os.path.join(HERE, "files.npz"), **out)
    print("files: done", len(msgs), "messages")


def make_methods():
    """SYM / ACIQ / GSS / TABLE (clipping.py:51-139) end to end: packed bytes, per-row ranges
    and GSS loss_evals from the reference, on varied tables incl. edge rows."""
    rng = np.random.default_rng(23)
    tables = {
        "gauss64": gaussian_rows(501, 200, 64),
        "lap64": laplacian_rows(502, 100, 64, 0.3),
        "mixed17": mixed_table(150, 17, 503),
        "mixed128": mixed_table(60, 128, 504),
    }
    e = rng.standard_normal((12, 9)).astype(np.float32)
    e[0] = 0.0
    e[1] = 3.25
    e[2] = -np.abs(e[2])
    e[3] *= 1e-30
    e[4] *= 1e30
    e[5, :] = [0, 0, 0, 0, 0, 0, 0, 0, 1e-3]
    e[6] = -0.0
    tables["edge9"] = e
    tables["d1"] = rng.standard_normal((7, 1)).astype(np.float32)
    tables["d2"] = rng.standard_normal((7, 2)).astype(np.float32)
    out = {}
    for tname, x in tables.items():
        out[f"x_{tname}"] = x
        t = eq.EmbeddingTable(x)
        for method in ("sym", "aciq", "gss", "table"):
            for aux in ("fp16", "fp32"):
                q = eq.quantize_table(t, method, 4, aux)
                out[f"packed_{tname}_{method}_{aux}"] = eq.pack_table4(q).buffer.copy()
            if method == "table":
                cr = eq.clip_range_table(t)
                out[f"range_{tname}_table"] = np.array([cr.xmin, cr.xmax])
                continue
            lo, hi, ev = [], [], []
            for i in range(t.rows):
                c = eq.WorkCounters()
                cr = eq.row_clip_range(method, t.row(i), 4, counters=c)
                lo.append(cr.xmin); hi.append(cr.xmax); ev.append(c.loss_evals)
            out[f"range_{tname}_{method}"] = np.array([lo, hi])
            out[f"evals_{tname}_{method}"] = np.array(ev, np.int64)
    np.savez_compressed(os.path.join(HERE, "methods.npz"), **out)
    print("methods: done", len(tables), "tables")


def make_kmeans():
    """Row-wise KMEANS codebooks (codebook.py:35-172) and its EMBQ container from the reference."""
    import tempfile

    from embquant import fileio

    rng = np.random.default_rng(31)
    tables = {
        "gauss64": gaussian_rows(601, 120, 64),
        "lap64": laplacian_rows(602, 60, 64, 0.5),
        "mixed17": mixed_table(80, 17, 603),
        "mixed200": mixed_table(20, 200, 604),
    }
    e = rng.standard_normal((10, 20)).astype(np.float32)
    e[0] = 0.0
    e[1] = np.arange(20) % 5
    e[2] = np.arange(20) % 16
    e[3] = np.arange(20) % 17
    e[4] *= 1e-25
    e[5, :10] = 1.0
    tables["edge20"] = e
    tables["d1"] = rng.standard_normal((5, 1)).astype(np.float32)
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for tname, x in tables.items():
            out[f"x_{tname}"] = x
            for aux in ("fp16", "fp32"):
                q = eq.quantize_table(eq.EmbeddingTable(x), "kmeans", 4, aux)
                out[f"books_{tname}_{aux}"] = np.ascontiguousarray(q.codebooks)
                out[f"idx_{tname}_{aux}"] = np.ascontiguousarray(q.indices)
                path = os.path.join(tmp, "k.embq")
                fileio.write_embq(path, q)
                out[f"embq_{tname}_{aux}"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "kmeans.npz"), **out)
    print("kmeans: done", len(tables), "tables")


def make_hist_apprx():
    """HIST-APPRX windows (histclip.py:181-217) from the reference.  Its norms go through
    numpy's SIMD pow and are host-dependent in the last bit, so only the windows, ranges and
    packed rows are recorded."""
    tables = {"gauss64": gaussian_rows(701, 150, 64), "lap64": laplacian_rows(702, 100, 64, 0.4),
              "mixed33": mixed_table(100, 33, 703)}
    out = {}
    for tname, x in tables.items():
        out[f"x_{tname}"] = x
        for b in (200, 40, 8):
            st, ns, lo, hi = [], [], [], []
            for row in x:
                h = eq.hist_apprx_search(row, b)
                st.append(h.start_bin); ns.append(h.nbins_selected)
                lo.append(h.clip_range.xmin); hi.append(h.clip_range.xmax)
            out[f"win_{tname}_{b}"] = np.array([st, ns])
            out[f"range_{tname}_{b}"] = np.array([lo, hi])
        q = eq.quantize_table(eq.EmbeddingTable(x), "hist-apprx", 4, "fp16")
        out[f"packed_{tname}"] = eq.pack_table4(q).buffer.copy()
    np.savez_compressed(os.path.join(HERE, "hist_apprx.npz"), **out)
    print("hist_apprx: done")


def signed_zero_rows(d, rng):
    """Rows whose min or max is a zero: numpy's np.min / np.max then return one of several
    equal extrema, and that choice is the sign of the packed bias (uniform.py:80)."""
    rows = []
    for kind in range(6):
        for _ in range(6):
            x = (np.abs(rng.standard_normal(d)) + 0.01).astype(np.float32)
            nz = int(rng.integers(1, max(1, min(d, 6)) + 1))
            pos = rng.choice(d, nz, replace=False)
            if kind == 0:      # lone -0.0 minimum
                x[pos[0]] = -0.0
            elif kind == 1:    # +0.0 / -0.0 minimum ties
                x[pos] = np.where(rng.random(nz) < 0.5, np.float32(0.0), np.float32(-0.0))
            elif kind == 2:    # all zeros of random signs
                x[:] = np.where(rng.random(d) < 0.5, np.float32(0.0), np.float32(-0.0))
            elif kind == 3:    # zero maximum (negative row), mixed signs
                x = -x
                x[pos] = np.where(rng.random(nz) < 0.5, np.float32(0.0), np.float32(-0.0))
            elif kind == 4:    # lone -0.0 maximum
                x = -x
                x[pos[0]] = -0.0
            else:              # many zeros of both signs among positives
                k = max(1, d // 3)
                p2 = rng.choice(d, k, replace=False)
                x[p2] = np.where(rng.random(k) < 0.5, np.float32(0.0), np.float32(-0.0))
            rows.append(x)
    return np.stack(rows)


def make_signed_zero():
    """Every row-wise method on rows whose extremum is a (signed) zero: packed bytes and the
    float64 ranges with their zero signs, from the reference (np.min/np.max order, the
    greedy pair recording x0 + 0*step, histclip.py:170's lo + w*s)."""
    rng = np.random.default_rng(1911)
    out = {}
    for d in (1, 2, 7, 8, 9, 16, 17, 64, 65, 100, 128, 200, 300):
        x = signed_zero_rows(d, rng)
        out[f"x_{d}"] = x
        t = eq.EmbeddingTable(x)
        for method in ("asym", "sym", "greedy", "hist-brute", "hist-apprx", "aciq", "gss"):
            b = 40 if method == "hist-brute" and d > 64 else 200
            for aux in ("fp16", "fp32"):
                q = eq.quantize_table(t, method, 4, aux, b=b)
                out[f"packed_{d}_{method}_{aux}"] = eq.pack_table4(q).buffer.copy()
            lo, hi = [], []
            for i in range(t.rows):
                cr = eq.row_clip_range(method, t.row(i), 4, b=b)
                lo.append(cr.xmin); hi.append(cr.xmax)
            out[f"range_{d}_{method}"] = np.array([lo, hi])
    np.savez_compressed(os.path.join(HERE, "signed_zero.npz"), **out)
    print("signed_zero: done")


if __name__ == "__main__":
    which = sys.argv[2:] or ["mse", "edge", "hist", "config1", "sls", "files", "methods", "kmeans",
                             "hist_apprx", "signed_zero"]
    for w in which:
        {"mse": make_mse, "edge": make_edge, "hist": make_hist, "config1": make_config1,
         "sls": make_sls, "files": make_files, "methods": make_methods, "kmeans": make_kmeans,
         "hist_apprx": make_hist_apprx, "signed_zero": make_signed_zero}[w]()
