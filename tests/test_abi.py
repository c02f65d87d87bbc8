"""The C-ABI library builds, loads and exports exactly what include/skc.h declares (CPU only)."""

import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "skc.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*|size_t)\s*\*?\s*(skc_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "skc_chain_fwd" in names and "skc_fit_run" in names and len(names) >= 10


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2512_04556_b200 import _build, _native
    lib_path = _build.build()
    lib = _native.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_native.EXPORTS)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (skc_\w+)", nm))
    assert set(declared_symbols()) <= exported
    assert lib.skc_version() == 200
    assert lib.skc_max_taps() >= 128


def test_sm100a_cubin_in_library():
    from paper_2512_04556_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_build.LIB)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_bad_arguments_fail_without_a_device():
    """Argument validation happens before any CUDA call."""
    import ctypes
    import numpy as np
    from paper_2512_04556_b200 import _native as nat
    lib = nat.load_library()
    taps = np.zeros((1, 3))
    rc = lib.skc_layer_fwd(None, 0, None, 0, 1, 4, 4, 3, nat.dbl(taps), 1, 0, None)
    assert rc == nat.SKC_EBADARG
    assert b"null" in lib.skc_last_error()
    rc = lib.skc_layer_fwd(ctypes.c_void_p(16), 0, ctypes.c_void_p(16), 0, 1, 4, 4, 7, nat.dbl(taps), 1, 0, None)
    assert rc == nat.SKC_EBADARG


def test_sparse_stencil_compiles_without_a_device(tmp_path, monkeypatch):
    """The generated sparse stencil of config 1's wide layers compiles with
    NVRTC for sm_100a (no device needed), for every input/output variant."""
    import numpy as np
    from paper_2512_04556_b200 import _native as nat
    from paper_2512_04556_b200 import synth
    lib = nat.load_library()
    cpx = synth.c1_complex()
    t = np.ascontiguousarray(cpx.layers[0].taps())
    assert lib.skc_sparse_compile_check(nat.dbl(t), t.shape[0], nat.SKC_F32, nat.SKC_CHW, nat.SKC_F32, nat.SKC_CHW) == 1
    t = np.ascontiguousarray(cpx.layers[2].taps())
    for args in ((nat.SKC_F32, nat.SKC_CHW, nat.SKC_F32, nat.SKC_CHW), (nat.SKC_F16, nat.SKC_CHW, nat.SKC_F16, nat.SKC_HWC),
                 (nat.SKC_F32, nat.SKC_HWC, nat.SKC_F32, nat.SKC_CHW)):
        rc = lib.skc_sparse_compile_check(nat.dbl(t), t.shape[0], *args)
        assert rc == 0, nat.last_error()
    # all-channel chain heads (HWC in, planar out): config 1's fp32 D5 head and
    # config 3's fp16 Kawase head (dense-size layers the generator takes as heads)
    for layer, dt in ((cpx.layers[0], nat.SKC_F32), (synth.kawase_complex().layers[0], nat.SKC_F16)):
        t = np.ascontiguousarray(layer.taps())
        rc = lib.skc_sparse_compile_check(nat.dbl(t), t.shape[0], dt, nat.SKC_HWC, dt, nat.SKC_CHW)
        assert rc == 0, nat.last_error()


def test_layer_routing_of_the_benchmark_complexes():
    """skc_layer_plan (no device needed) routes config 1's wide layers to the
    generated sparse stencil (kind 3, merged position counts 58 / 102 / 116),
    its 5 x 5 head to the dense kernel (kind 1, D = 5: on HWC input it runs as
    the all-channel generated head), and config 3's 4-tap Kawase layers to
    the tap kernel (kind 0)."""
    import ctypes
    import numpy as np
    from paper_2512_04556_b200 import _native as nat
    from paper_2512_04556_b200 import synth
    lib = nat.load_library()

    def plan(layer, c):
        t = np.ascontiguousarray(layer.taps())
        k, p = ctypes.c_int(), ctypes.c_int()
        assert lib.skc_layer_plan(nat.dbl(t), t.shape[0], 2665, 1264, c, 0, ctypes.byref(k), ctypes.byref(p)) == 0
        return k.value, p.value

    assert [plan(l, 3) for l in synth.c1_complex().layers] == [(1, 5), (3, 58), (3, 102), (3, 116)]
    kaw = [plan(l, 4) for l in synth.kawase_complex().layers]
    assert kaw[0] == (1, 3) and all(k == 0 for k, _ in kaw[1:])
    t = np.ascontiguousarray(synth.c1_complex().taps())
    lay = np.ascontiguousarray(synth.c1_complex().layout, dtype=np.int32)
    # fp32 chain: no input relayout (the head reads HWC), no output relayout (staged epilogue)
    assert lib.skc_chain_relayouts(nat.dbl(t), nat.ints(lay), 4, 2665, 1264, 3, nat.SKC_F32, 0) == 0
    tk = np.ascontiguousarray(synth.kawase_complex().taps())
    lk = np.ascontiguousarray(synth.kawase_complex().layout, dtype=np.int32)
    # fp16 Kawase chain: the all-channel fp16 head replaces the input relayout pass
    assert lib.skc_chain_relayouts(nat.dbl(tk), nat.ints(lk), 6, 2160, 3840, 4, nat.SKC_F16, 0) == 0
    assert lib.skc_chain_mid_dtype(nat.ints(lk), 6, nat.SKC_F16, nat.SKC_F16) == nat.SKC_F16


def test_pair_compiles_without_a_device():
    """The fused head pair (layers 0+1 in one launch, skc_layer_pair_fwd) of
    configs 0 and 1 compiles with NVRTC for sm_100a; a pair whose second layer
    is taller than the streamed block is declined (SKC_ENOTTAKEN)."""
    import numpy as np
    from paper_2512_04556_b200 import _native as nat
    from paper_2512_04556_b200 import synth
    lib = nat.load_library()
    for cpx in (synth.c1_complex(), synth.c0_complex()):
        t0, t1 = (np.ascontiguousarray(l.taps()) for l in cpx.layers[:2])
        rc = lib.skc_pair_compile_check(nat.dbl(t0), t0.shape[0], nat.dbl(t1), t1.shape[0])
        assert rc == nat.SKC_OK, nat.last_error()
    # a second layer taller than the streamed block (reach 40 rows) is declined
    t0 = np.ascontiguousarray(synth.c1_complex().layers[0].taps())
    tall = np.array([[0.25, -40.5, 0.5], [-0.75, 40.25, 0.5]], dtype=np.float64)
    assert lib.skc_pair_compile_check(nat.dbl(t0), t0.shape[0], nat.dbl(tall), tall.shape[0]) == nat.SKC_ENOTTAKEN
