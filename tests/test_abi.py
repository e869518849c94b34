"""CPU checks of the C-ABI library: it loads, exports every symbol include/oica.h declares,
maps statuses, refuses non-sm_100 / absent devices, and its host-only selection merge
(reading A6) decides as the oracle's selection rule does."""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from paper_2408_17118_b200 import oica

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "oica.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(oica_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = oica.lib()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(oica.SIGNATURES), set(names) ^ set(oica.SIGNATURES)


def test_library_is_sm100a_binary():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", oica.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    for k, name in enumerate(oica.STATUS):
        assert oica.lib().oica_status_string(k).decode() == "OICA_" + ("OK" if k == 0 else "ERR_" + name)


def test_create_without_device_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(oica.OicaError) as e:
        oica.Context(device=0)
    assert e.value.name in ("CUDA", "UNSUPPORTED_DEVICE")


def test_nccl_is_loadable_and_makes_unique_ids():
    """The L/M-shard exchange dlopens NCCL; ncclGetUniqueId needs no GPU."""
    a, b = oica.nccl_unique_id(), oica.nccl_unique_id()
    assert len(a) == 128 and a != b


def _unit(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v)


def test_merge_records_cluster_rule():
    a, b = _unit([1, 2, 0.5]), _unit([-1, 0.3, 2])
    W = np.array([a, b, -a, a + 1e-6 * b, b])
    W /= np.linalg.norm(W, axis=1, keepdims=True)
    recs = [dict(upsilon=1.0, alpha=1.5, q=30, size=5),
            dict(upsilon=0.9, alpha=1.2, q=3, size=2),
            dict(upsilon=1.0 + 1e-9, alpha=1.5, q=12, size=7),
            dict(upsilon=1.0 - 1e-9, alpha=1.5, q=40, size=1),
            dict(upsilon=0.9, alpha=1.2, q=8, size=4, valid=0)]
    r = oica.merge_records(recs, W)
    assert r["status"] == 0 and r["winner"] == 2 and r["size"] == 13 and not r["near_tie"]
    # a tie between two different fixed points -> near_tie, lowest q wins
    recs[1]["upsilon"] = 1.0 + 1e-9
    r = oica.merge_records(recs, W)
    assert r["near_tie"] and r["winner"] == 1
    assert oica.merge_records([dict(upsilon=1, alpha=1, q=0, size=1, valid=0)], W[:1])["status"] != 0


@pytest.mark.parametrize("N,k", [(5, 0), (5, 2), (12, 7), (64, 1), (256, 31), (256, 255)])
def test_complement_basis_host(N, k):
    """OICA_REDUCE_X basis: rows orthonormal, orthogonal to W, and G^T G = I - W^T W
    (the projection of Alg. 1, so b0 = G r/||G r|| starts the same trajectory as P r/||P r||, A9)."""
    rs = np.random.default_rng(N * 100 + k)
    W = np.linalg.qr(rs.standard_normal((N, max(k, 1))))[0][:, :k].T if k else np.zeros((0, N))
    G = oica.complement_basis(W, N)
    assert G.shape == (N - k, N)
    assert np.abs(G @ G.T - np.eye(N - k)).max() < 1e-12
    if k:
        assert np.abs(G @ W.T).max() < 1e-12
    assert np.abs(G.T @ G - (np.eye(N) - W.T @ W)).max() < 1e-12


@pytest.mark.parametrize("N,d", [(6, 6), (6, 3), (40, 33), (256, 225)])
def test_deflate_basis_host(N, d):
    """One accepted row: the new basis spans exactly span(G) minus w = G^T b (Alg. 2 line 28)."""
    rs = np.random.default_rng(N + d)
    G = np.linalg.qr(rs.standard_normal((N, d)))[0].T               # d x N, orthonormal rows
    b = rs.standard_normal(d)
    b /= np.linalg.norm(b)
    w = G.T @ b
    G2 = oica.deflate_basis(G, b)
    assert G2.shape == (d - 1, N)
    assert np.abs(G2 @ G2.T - np.eye(d - 1)).max() < 1e-12
    assert np.abs(G2 @ w).max() < 1e-12
    # inside span(G): projecting onto span(G) changes nothing
    assert np.abs(G2 - (G2 @ G.T) @ G).max() < 1e-12
    # G2^T G2 = G^T G - w w^T
    assert np.abs(G2.T @ G2 - (G.T @ G - np.outer(w, w))).max() < 1e-12


def test_split_parts_host():
    """Split-slot parts: a function of (global active count, S); never more work units than the
    launch grid provides (tiles x P <= 296 / S whenever P > 1), non-decreasing as runs leave,
    and 1 once the row tiles alone fill the GPU."""
    for S in (1, 2, 7, 30, 61, 128):
        prev = None
        for L in list(range(1, 600)) + [1000, 2048, 4096, 16384, 65536]:
            P = oica.split_parts(L, S)
            tiles2 = -(-(-(-L // 128)) // 2) * 2
            assert 1 <= P <= 8
            if P > 1:
                assert tiles2 * S <= 148 and tiles2 * S * P <= 296
            else:
                assert tiles2 * S > 148 or 296 // (tiles2 * S) <= 1
            if prev is not None:
                assert P <= prev
            prev = P
    with pytest.raises(oica.OicaError):
        oica.split_parts(10, 0)


@pytest.mark.parametrize("M", [1, 2000, 5003, 20000, 150001, 250000, 1_000_000, 4_000_000, 40_000_000])
def test_slot_plan_host(M):
    """Slots (the fixed fp32-accumulation units of every row): a function of the global M and the
    precision only, a multiple of the kernel chunk widths (tensor cores: 384; FP32 at small M: 64),
    covering M; an M-sharded rank's slots have the same length and cover its samples."""
    for prec in (oica.PREC_TC, oica.PREC_FP32, oica.PREC_AUTO):
        ln, S = oica.slot_plan(M, precision=prec)
        fp32 = prec == oica.PREC_FP32 or (prec == oica.PREC_AUTO and M < 16384)
        short = fp32 and M < 65536
        align = 64 if short else 384
        assert ln % align == 0 and 1 <= S <= 128 and (S - 1) * ln < M <= S * ln, (prec, ln, S)
        if short:   # slots of >= 128 samples, up to 128 of them: many CTAs for few row tiles
            n_s = min(128, -(-M // 128))
            assert ln == 64 * -(-(-(-M // n_s)) // 64), (M, ln)
        for world in (2, 8):
            ml = -(-M // world)
            ln2, S2 = oica.slot_plan(M, min(ml, M), precision=prec)
            assert ln2 == ln and (S2 - 1) * ln2 < min(ml, M) <= S2 * ln2


def test_bench_refuses_experiment_variables():
    env = dict(os.environ, OICA_TC_EPI="3")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "cfg0_tiny"], capture_output=True,
                         text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 2 and "OICA_TC_EPI" in out.stderr and not out.stdout.strip()
