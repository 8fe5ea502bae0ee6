"""EMBT / EMBQ containers (fileio.py) against bytes and messages from the reference
(tests/golden/files.npz); the streamed EMBT -> EMBQ pipeline on the GPU."""

import json
import os

import numpy as np
import pytest

import oracle
import paper_1911_02079_b200 as eq

G = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    return np.load(os.path.join(G, "files.npz"))


def test_write_embt_bytes_match_reference(tmp_path):
    f = _golden()
    p = tmp_path / "t.embt"
    eq.write_embt(p, f["table"])
    assert p.read_bytes() == f["embt"].tobytes()
    t = eq.read_embt(p)
    assert np.array_equal(t.values, f["table"])


def test_read_errors_match_reference(tmp_path):
    f = _golden()
    msgs = json.loads(str(f["messages"]))
    for k, want in msgs.items():
        p = tmp_path / k
        p.write_bytes(f["bad_" + k].tobytes())
        reader = eq.read_embt if k.startswith("embt") else eq.read_embq
        with pytest.raises(eq.DataError) as e:
            reader(str(p))
        assert str(e.value).replace(str(tmp_path), "<dir>") == want, k


def test_read_embq_and_host_write_embq_roundtrip(tmp_path):
    f = _golden()
    for name in ("greedy_fp16", "asym_fp32", "hist_fp16"):
        src = tmp_path / (name + ".embq")
        src.write_bytes(f["embq_" + name].tobytes())
        p = eq.read_embq(src)
        assert p.rows == 37 and p.dim == 9
        assert p.aux_precision == name.split("_")[1]
        dst = tmp_path / (name + "_copy.embq")
        eq.write_embq(dst, p)   # host buffer through the native writer
        assert dst.read_bytes() == src.read_bytes()


def test_off_path_schemes_and_methods_raise(tmp_path):
    f = _golden()
    blob = bytearray(f["embq_greedy_fp16"].tobytes())
    blob[8] = 1   # uniform8
    p = tmp_path / "u8.embq"
    p.write_bytes(bytes(blob))
    with pytest.raises(ValueError, match="not on the B200 hot path"):
        eq.read_embq(p)
    t = tmp_path / "t.embt"
    t.write_bytes(f["embt"].tobytes())
    with pytest.raises(ValueError, match="not on the B200 hot path"):
        eq.quantize_file(t, tmp_path / "o.embq", "kmeans-cls")
    with pytest.raises(ValueError, match="unknown method"):
        eq.quantize_file(t, tmp_path / "o.embq", "nope")
    with pytest.raises(ValueError, match=r"r must be in \(0, 1\]"):
        eq.quantize_file(t, tmp_path / "o.embq", "greedy", r=0.0)
    bad = tmp_path / "bad.embt"
    bad.write_bytes(f["bad_embt_magic"].tobytes())
    with pytest.raises(eq.DataError, match="bad magic b'EMBX'"):
        eq.quantize_file(bad, tmp_path / "o.embq", "greedy")
    assert not (tmp_path / "o.embq").exists()


@pytest.mark.gpu
def test_quantize_file_matches_reference_containers(tmp_path):
    f = _golden()
    src = tmp_path / "t.embt"
    src.write_bytes(f["embt"].tobytes())
    for name, method, aux in (("greedy_fp16", "greedy", "fp16"), ("asym_fp32", "asym", "fp32"),
                              ("hist_fp16", "hist-brute", "fp16")):
        out = tmp_path / (name + ".embq")
        eq.quantize_file(src, out, method, aux)
        assert out.read_bytes() == f["embq_" + name].tobytes(), name


@pytest.mark.gpu
@pytest.mark.parametrize("d,chunk", [(64, 4096), (17, 1000), (128, 0)])
def test_quantize_file_streams_chunks(tmp_path, d, chunk):
    from oracle import rng

    rows = 50_003
    x = rng.mixed_table(rows, d, 5)
    src = tmp_path / "big.embt"
    eq.write_embt(src, x)
    out = tmp_path / "big.embq"
    eq.quantize_file(src, out, "greedy", "fp16", chunk_rows=chunk)
    want = oracle.quantize_pack_table(x, "greedy", 200, 0.16, "fp16").packed
    blob = out.read_bytes()
    assert blob[:4] == b"EMBQ" and len(blob) == 26 + want.size
    assert blob[26:] == want.tobytes()
    p = eq.read_embq(out)
    assert (p.rows, p.dim, p.aux_precision) == (rows, d, "fp16")


@pytest.mark.gpu
def test_quantize_file_nonfinite_leaves_no_output(tmp_path):
    x = np.random.default_rng(1).standard_normal((9000, 32)).astype(np.float32)
    src = tmp_path / "t.embt"
    eq.write_embt(src, x)
    blob = bytearray(src.read_bytes())
    blob[25 + 4 * (7000 * 32 + 5):25 + 4 * (7000 * 32 + 6)] = np.array([np.inf], "<f4").tobytes()
    src.write_bytes(bytes(blob))
    out = tmp_path / "o.embq"
    with pytest.raises(eq.DataError, match="payload contains non-finite values"):
        eq.quantize_file(src, out, "greedy", chunk_rows=1024)
    assert not out.exists()


@pytest.mark.gpu
def test_write_embq_from_device_streams_hbm(tmp_path):
    import torch

    x = torch.randn(300_001, 64, device="cuda")
    p, _ = eq.quantize_pack_table4(x, "asym", "fp16")
    dev = tmp_path / "dev.embq"
    eq.write_embq(dev, p)          # device buffer, chunked D2H + write
    host = tmp_path / "host.embq"
    eq.write_embq(host, eq.PackedTable4(p.rows, p.dim, "fp16", buffer=p.device_buffer.cpu().numpy()))
    assert dev.read_bytes() == host.read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["table", "sym", "gss", "hist-apprx"])
def test_quantize_file_other_methods_span_chunks(tmp_path, method):
    """TABLE's single range must cover the whole file, not each streamed chunk."""
    from oracle import rng

    x = rng.mixed_table(9000, 24, 3)
    x[8500] *= 50.0                      # the table extremes sit in the last chunk
    src = tmp_path / "t.embt"
    eq.write_embt(src, x)
    out = tmp_path / "t.embq"
    eq.quantize_file(src, out, method, "fp32", chunk_rows=1000)
    want = oracle.quantize_pack_table(x, method, 200, 0.16, "fp32").packed
    assert out.read_bytes()[26:] == want.tobytes()


@pytest.mark.gpu
def test_quantize_file_kmeans_matches_reference_container(tmp_path):
    f = np.load(os.path.join(G, "kmeans.npz"))
    x = f["x_gauss64"]
    src = tmp_path / "k.embt"
    eq.write_embt(src, x)
    out = tmp_path / "k.embq"
    eq.quantize_file(src, out, "kmeans", "fp16")
    assert out.read_bytes() == f["embq_gauss64_fp16"].tobytes()
