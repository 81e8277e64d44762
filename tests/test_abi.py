"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every
symbol include/vlq_gpu.h declares, and the Python surface mirrors the
reference's vlqadc module (names, defaults).  No compute calls (no GPU)."""
import ctypes
import inspect
import os

import numpy as np
import pytest

from conftest import ROOT


def test_library_exports_every_header_symbol():
    from paper_1901_00275_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _lib.header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and every header function has a ctypes signature in the binding
    assert set(names) == set(_lib._SIGS)


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1901_00275_b200", "libvlqgpu.so")
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_python_surface_mirrors_reference():
    from paper_1901_00275_b200 import vlqadc
    # bindings.cpp:207-221 / __init__.py:8-24
    for name in ["Index", "brute_force_gt", "gen_synthetic", "read_vecs", "set_max_threads", "write_vecs"]:
        assert hasattr(vlqadc, name)
    sig = inspect.signature(vlqadc.Index.train)
    assert list(sig.parameters)[:7] == ["train", "k", "n", "m", "iters", "seed", "clamp_lambda"]
    assert [sig.parameters[p].default for p in ["k", "n", "m", "iters", "seed", "clamp_lambda"]] == \
        [1024, 16, 8, 10, 42, True]
    sig = inspect.signature(vlqadc.Index.search)
    assert list(sig.parameters)[:5] == ["self", "queries", "w1", "alpha", "k"]
    assert [sig.parameters[p].default for p in ["w1", "alpha", "k"]] == [64, 0.25, 10]
    sig = inspect.signature(vlqadc.gen_synthetic)
    assert [sig.parameters[p].default for p in ["clusters", "spread", "seed"]] == [200, 0.05, 42]
    for prop in ["k", "n", "m", "dim", "ntotal"]:
        assert isinstance(getattr(vlqadc.Index, prop), property)


def test_gen_synthetic_is_bit_identical_to_reference():
    """Host-side generator; the stream must equal dataset.cpp:13-44."""
    from paper_1901_00275_b200 import vlqadc
    from conftest import load_golden
    z, _, _ = load_golden("smoke")
    a = vlqadc.gen_synthetic(5000, 16, clusters=20, spread=0.05, seed=42)
    assert np.array_equal(a[:64], z["base_head"])
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "vlqadc")):
        import subprocess
        import sys
        code = ("import sys,numpy as np; sys.path.insert(0, %r); import vlqadc;"
                "np.save(sys.argv[1], vlqadc.gen_synthetic(777, 7, clusters=5, spread=0.3, seed=9))" % ref)
        out = os.path.join("/tmp", f"gs_{os.getpid()}.npy")
        subprocess.run([sys.executable, "-c", code, out], check=True)
        assert np.array_equal(np.load(out), vlqadc.gen_synthetic(777, 7, clusters=5, spread=0.3, seed=9))
        os.remove(out)


def test_gen_synthetic_errors():
    from paper_1901_00275_b200 import vlqadc
    with pytest.raises(RuntimeError, match="dim and clusters must be positive"):
        vlqadc.gen_synthetic(10, 0)
    with pytest.raises(RuntimeError, match="spread must be positive"):
        vlqadc.gen_synthetic(10, 4, spread=0.0)


def test_vecs_roundtrip(tmp_path):
    # test_smoke.py:80-85 and the .bvecs/.ivecs widening (vecs_io.cpp:62-77)
    from paper_1901_00275_b200 import vlqadc
    a = vlqadc.gen_synthetic(50, 8, seed=3)
    p = str(tmp_path / "a.fvecs")
    vlqadc.write_vecs(a, p)
    assert np.array_equal(vlqadc.read_vecs(p), a)
    b = np.arange(40, dtype=np.float32).reshape(5, 8)
    for ext in ("bvecs", "ivecs"):
        p = str(tmp_path / f"b.{ext}")
        vlqadc.write_vecs(b, p)
        assert np.array_equal(vlqadc.read_vecs(p), b)
    with pytest.raises(RuntimeError, match="not representable as byte"):
        vlqadc.write_vecs(b + 0.5, str(tmp_path / "c.bvecs"))
    with pytest.raises(RuntimeError, match="cannot open"):
        vlqadc.read_vecs(str(tmp_path / "missing.fvecs"))


def test_code_bank_relabeling_is_a_balanced_permutation():
    """Host logic of the fast scan's code relabeling (engine.cu
    choose_code_banks): every sub-space's map is a permutation of 0..255 with
    8 values per bank (v mod 32), and values that always occur together --
    planted here as 32 groups of 8 -- are spread over 8 different banks."""
    from paper_1901_00275_b200 import _lib
    lib = _lib.lib()
    m = 3
    rng = np.random.default_rng(0)
    cooc = np.zeros((m, 256, 256), np.uint32)
    groups = [rng.permutation(256).reshape(32, 8) for _ in range(m)]
    for p in range(m):
        noise = rng.integers(0, 3, (256, 256)).astype(np.uint32)
        cooc[p] = np.triu(noise, 1)
        for g in groups[p]:
            for i in range(8):
                for j in range(i + 1, 8):
                    a, b = sorted((int(g[i]), int(g[j])))
                    cooc[p, a, b] += 1000
        cooc[p][np.arange(256), np.arange(256)] = 500
    perm = np.zeros((m, 256), np.uint8)
    assert lib.vlq_code_banks(cooc.ctypes.data, m, perm.ctypes.data) == 0
    for p in range(m):
        assert sorted(perm[p].tolist()) == list(range(256))
        assert np.array_equal(np.bincount(perm[p] % 32, minlength=32), np.full(32, 8))
        for g in groups[p]:
            assert len(set((perm[p][g] % 32).tolist())) == 8, (p, g)
    assert lib.vlq_code_banks(None, 1, perm.ctypes.data) != 0
