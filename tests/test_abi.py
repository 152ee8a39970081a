"""CPU-side checks of the C ABI: the library loads, exports exactly what
include/scrooge_b200.h declares, validates configs like AlignerConfig::validate
(proj/src/aligner.cpp:8-18) and refuses to compute without a GPU (no CPU
fallback). Host-only helpers (packing, synthetic pairs) run here too."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scrooge_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(sg):
    from paper_2208_09985_b200 import _ffi
    lib = C.CDLL(_ffi.LIB_PATH)
    decl = declared_functions()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_ffi.EXPORTS) == decl


def test_library_is_built_for_sm100a(sg):
    from paper_2208_09985_b200 import _ffi
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _ffi.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("W,O,ok", [(64, 33, True), (64, 24, True), (1, 0, True), (128, 127, True),
                                    (129, 64, True), (1024, 1023, True), (1025, 0, False),
                                    (32, 32, False), (0, 0, False), (64, -1, False),
                                    (2000, 5, False)])
def test_config_validation(sg, W, O, ok):
    cfg = sg.AlignerConfig(W=W, O=O)
    if ok:
        cfg.validate()
    else:
        with pytest.raises(sg.ConfigError):
            cfg.validate()


def test_single_window_with_dent_is_a_config_error(sg):
    # aligner.cpp:14-15
    with pytest.raises(sg.ConfigError, match="trimmed table storage"):
        sg.AlignerConfig(mode="single", dent=True).validate()


def test_empty_sequence_is_an_input_error(sg):
    with pytest.raises(sg.InputError, match="empty"):
        sg.align("", "ACGT")
    with pytest.raises(sg.InputError, match="pair 'x': empty sequence"):
        sg.run_batch([sg.SeqPairRecord("x", "ACGT", "")])


def test_compute_fails_loudly_without_gpu(sg):
    from paper_2208_09985_b200 import _ffi
    if _ffi.load().sg_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(sg.CudaError, match="no CPU fallback"):
        sg.align("ACGT", "ACGA")


def test_pack_layout_matches_reference_codes(sg):
    rng = np.random.default_rng(5)
    texts = [rng.integers(0, 5, size=int(rng.integers(1, 200)), dtype=np.uint8).tobytes()
             for _ in range(50)]
    pats = [rng.integers(0, 4, size=int(rng.integers(1, 200)), dtype=np.uint8).tobytes()
            for _ in range(50)]
    codes = sg.CodesBatch.from_lists(texts, pats)
    pk = sg.pack(codes)
    p = pk.c
    words = np.ctypeslib.as_array(C.cast(p.seq, C.POINTER(C.c_uint32)), (p.seq_words,))
    nmask = np.ctypeslib.as_array(C.cast(p.nmask, C.POINTER(C.c_uint32)),
                                  ((p.seq_words * 16 + 31) // 32,))
    toff = np.ctypeslib.as_array(C.cast(p.text_off, C.POINTER(C.c_int64)), (50,))
    poff = np.ctypeslib.as_array(C.cast(p.pat_off, C.POINTER(C.c_int64)), (50,))

    def unpack(off, n):
        out = []
        for k in range(n):
            b = off + k
            c = (int(words[b >> 4]) >> (2 * (b & 15))) & 3
            if (int(nmask[b >> 5]) >> (b & 31)) & 1:
                c = 4
            out.append(c)
        return bytes(out)

    for k in range(50):
        assert toff[k] % 16 == 0 and poff[k] % 16 == 0
        assert unpack(int(toff[k]), len(texts[k])) == bytes(min(c, 4) for c in texts[k])
        assert unpack(int(poff[k]), len(pats[k])) == pats[k]


def test_synth_codes_match_oracle_generator(sg):
    import oracle_ffi as O
    for cfg in (1, 2, 3, 5):
        b = sg.synth_codes(cfg, 11, 4)
        spec = O.baseline_spec(cfg)
        for k in range(4):
            assert b.pair(k) == O.synth_pair(spec, 11 + k)


def test_synth_packed_equals_packed_codes(sg):
    a = sg.synth_packed(2, 0, 300)
    b = sg.pack(sg.synth_codes(2, 0, 300))
    wa = np.ctypeslib.as_array(C.cast(a.c.seq, C.POINTER(C.c_uint32)), (a.c.seq_words,))
    wb = np.ctypeslib.as_array(C.cast(b.c.seq, C.POINTER(C.c_uint32)), (b.c.seq_words,))
    assert a.c.seq_words == b.c.seq_words and (wa == wb).all()


def test_cigar_string_helpers(sg):
    assert sg.cigar_to_string([("=", 3), ("X", 1)]) == "3=1X"
    assert sg.cigar_from_string("3=1X2=3=") == [("=", 3), ("X", 1), ("=", 5)]
    with pytest.raises(sg.InputError):
        sg.cigar_from_string("3=0X")


def test_single_window_length_limits(sg):
    # aligner.cpp:92-94 through run_batch (batch.cpp:94-97): an input error naming the pair
    cfg = sg.AlignerConfig(mode="single", dent=False)
    with pytest.raises(sg.InputError, match="toolong.*at most 1024"):
        sg.run_batch([sg.SeqPairRecord("toolong", "A" * 2000, "A" * 2000)], cfg)
    # up to 1024 characters is valid (K6 on the GPU); without a device the call
    # fails as a CUDA error, never as a config error or a CPU fallback
    try:
        r = sg.run_batch([sg.SeqPairRecord("mid", "A" * 300, "A" * 299)], cfg)
        assert r.outcomes[0].found and r.outcomes[0].distance == 1
    except sg.CudaError:
        pass
    cfg.validate()  # single-window configs without DENT are valid


def test_first_bad_pair_of_a_large_batch(sg):
    """batch.cpp:18-25 names the first failing pair in input order. The length checks of a
    large batch run on the library's worker pool in chunks: the lowest index must still be
    the one reported, whichever chunk finds its bad pair first."""
    batch = sg.synth_packed(1, 0, 200000)
    tl, pl = batch.lengths()
    saved = (int(tl[150001]), int(pl[60002]), int(pl[199999]))
    try:
        tl[150001] = 0
        pl[60002] = 0
        pl[199999] = 0
        for _ in range(20):  # (any worker may reach its chunk's bad pair first)
            with pytest.raises(sg.InputError, match=r"pair '60002': empty sequence"):
                sg.align_packed(sg.AlignerConfig(W=64, O=24), batch)
    finally:
        tl[150001], pl[60002], pl[199999] = saved
