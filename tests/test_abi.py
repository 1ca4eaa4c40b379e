"""The C-ABI library (CPU side): it loads, exports every symbol include/me.h
declares, and its host-only logic (space size, decode) agrees with the oracle's
enumeration.  No compute call runs here (no GPU)."""
import re
import subprocess
from pathlib import Path

import pytest

import me_inputs as mi

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    txt = (ROOT / "include" / "me.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|uint64_t)\s+(me_\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def me():
    from paper_2411_06465_b200 import build
    build.build()
    import paper_2411_06465_b200 as me
    return me


def test_exports_every_declared_symbol(me):
    from paper_2411_06465_b200 import _abi
    decl = header_functions()
    assert len(decl) >= 20
    assert sorted(_abi.EXPORTS) == decl
    out = subprocess.check_output(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)], text=True)
    syms = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for name in decl:
        assert name in syms, name
        assert hasattr(_abi.lib(), name)


def test_library_is_sm100a(me):
    from paper_2411_06465_b200 import _abi
    out = subprocess.check_output(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], text=True)
    assert "sm_100a" in out


def test_compute_fails_loudly_without_gpu(me):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(me.MEError) as e:
        me.me_estimate(mi.PRESETS["llama3.1-8b"], d=1, t=1, p=1, c=1, b=1, s=8192)
    assert e.value.status == me._abi.ME_ECUDA


@pytest.mark.parametrize("name", ["C1", "C3", "C3u", "rand1", "rand2"])
def test_space_size_and_decode_match_oracle(me, oracle_mod, name):
    if name == "C3u":
        sp = mi.config("C3", uneven=1)
    elif name == "rand1":
        sp = mi.Space(models=mi.random_models(4, seed=11, small=True), world=[6, 12, 8], caps_gb=[1],
                      mbs=[1, 2, 3], seq=[8, 12, 16], gbs=48, uneven=1)
    elif name == "rand2":
        sp = mi.Space(models=mi.random_models(3, seed=12), world=mi.random_world_sizes(12), caps_gb=[40, 80],
                      mbs=[1, 4], seq=[4096, 6144], max_t=8, gpus_per_node=8, rc_mask=2, do_mask=1)
    else:
        sp = mi.config(name)
    n = oracle_mod.space_size(sp)
    assert me.me_space_size(sp) == n
    step = max(1, n // 61)
    for i in list(range(0, n, step)) + [n - 1]:
        assert me.me_decode(sp, i) == oracle_mod.decode(sp, i), i
    with pytest.raises(me.MEError):
        me.me_decode(sp, n)


def test_large_space_sizes(me, oracle_mod):
    for name in ("C4", "C5"):
        sp = mi.config(name)
        assert me.me_space_size(sp) == oracle_mod.space_size(sp)


def test_invalid_inputs(me):
    sp = mi.config("C1")
    bad = mi.Space(models=[(4096, 11008, 32, 32, 7, 32000)], world=[8], caps_gb=[80], mbs=[1], seq=[4096])
    with pytest.raises(me.MEError) as e:
        me.me_space_size(bad)
    assert e.value.status == me._abi.ME_EINVAL
    with pytest.raises(me.MEError):
        me.me_space_size(mi.Space(models=sp.models, world=[8], caps_gb=[1] * 9, mbs=[1], seq=[8]))
    with pytest.raises(me.MEError):
        me.me_space_size(mi.Space(models=sp.models, world=[8], caps_gb=[1], mbs=[1], seq=[8], rc_mask=0))


def test_digest_merge_matches_oracle(me, oracle_mod):
    """me_digest_merge (host-only): the digest of a result from its pieces'
    digests equals the oracle's digest of the whole (or_digest in one piece)"""
    import me_inputs as mi
    sp = mi.config("C3", uneven=1)
    whole = oracle_mod.digest(sp, chunk=1 << 40, threads=4)[0]
    parts = oracle_mod.digest(sp, chunk=7777, threads=4)
    got = me.digest_merge([int(r[0]) for r in parts], [(int(r[9]), int(r[10])) for r in parts])
    assert got == (int(whole[9]), int(whole[10]))
    assert me.digest_merge([], []) == (0, 0)
