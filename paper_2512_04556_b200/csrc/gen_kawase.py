"""Emit the pass bodies of the fused separable Kawase kernel (skc_kawase.cu)
for the instantiated ladders b_l = l, L = 1..6.

The passes are streaming 1-D filters with per-layer delay lines.  Written as
templated loops over arrays, nvcc's front end spent minutes unrolling them;
emitted here as named registers and blocks of P stream steps (the ring slots
and warm-up bounds resolved in Python), they compile in seconds.  _build.py
runs this before nvcc; the output lands in build/ (not tracked).
tools/kawase_gen_check.py runs the emitted H statements in Python against the
direct chain (tests/test_host.py).

    python gen_kawase.py OUT.inc
"""

from __future__ import annotations

import sys

TW = 128      # output columns per band (kKwTW)
R = 32        # rows per V iteration (kKwR)
HP2 = (TW * 4 + 2) // 2   # H-result row pitch in float2 (kKwHP / 2)
MAX_L = 6


def ladder(L):
    return [l for l in range(L)]


def lag(bs, l):
    return sum(b + 1 for b in bs[:l + 1])


def start(bs, l):
    return 2 * (lag(bs, l - 1) if l > 0 else 0)


P = 16    # loop period: every ring size divides it (ring_size), so slots are compile-time


def ring_size(D):
    r = 1
    while r < D:
        r *= 2
    assert P % r == 0
    return r


def h_loop_body(bs, tw):
    """Horizontal passes of one row segment of `tw` output columns as a
    rolled loop over blocks of P stream steps (skewed wavefront inside a
    block: at step tau layer l handles index tau - l).  Delay lines have a
    power-of-two size R_l >= 2 b_l + 1 dividing P, so every ring slot is a
    compile-time register within the block and the code is one block long
    (the fully unrolled row was ~100 KB of SASS: instruction-cache bound).
    State starts at zero: outputs before a layer's warm-up are never stored
    (a stored output only depends on inputs inside the row).  With EDGE, a
    block whose layer positions all lie inside the image (a per-block uniform
    test) runs without the per-step masks: only the 2-3 blocks next to the
    image edge pay for them."""
    L = len(bs)
    RX = lag(bs, L - 1)
    IW = tw + 2 * RX
    nblk = (IW + L - 1 + P - 1) // P
    Rs = [ring_size(2 * b + 1) for b in bs]
    regs = ["sv", "z2"] + [f"a{l}" for l in range(L + 1)] + [f"p{l}" for l in range(L)] + \
        [f"r{l}_{i}" for l in range(L) for i in range(Rs[l])]
    out = [f"    float2 {', '.join(regs)};",
           "    z2 = make_float2(0.f, 0.f);"]
    out.append("    " + " ".join(f"{r} = z2;" for r in regs[2:]))
    out.append(f"#pragma unroll 1")
    out.append(f"    for (int j = 0; j < {nblk}; ++j) {{")
    out.append(f"        const unsigned *inj = in + {2 * P} * j;")
    out.append(f"        const int kj = {P} * j;")

    def block(masked):
        for t in range(P):
            for l in reversed(range(L)):
                D = 2 * bs[l] + 1
                R = Rs[l]
                if l == 0:
                    out.append(f"        a0 = h2f2(inj[{2 * t}]);")
                rd = f"r{l}_{(t - l - D) % R}"
                wr = f"r{l}_{(t - l) % R}"
                out.append(f"        sv = add2(a{l}, p{l}); p{l} = a{l}; a{l + 1} = add2(sv, {rd}); {wr} = sv;")
                if masked:
                    out.append(f"        if ((unsigned)(xg0 + kj + {t - l - lag(bs, l)}) >= (unsigned)W) a{l + 1} = z2;")
                if l == L - 1:
                    o = t - (L - 1) - 2 * RX
                    out.append(f"        {{ const int oc = kj + {o}; if ((unsigned)oc < {tw}u) out[2 * oc] = a{L}; }}")

    lo = -(L - 1) - RX              # smallest / largest position offset a block's layer steps touch
    hi = P - 1 - lag(bs, 0)
    out.append(f"        if (EDGE && (xg0 + kj + {lo} < 0 || xg0 + kj + {hi} >= W)) {{")
    block(True)
    out.append("        } else {")
    block(False)
    out.append("        }")
    out.append("    }")
    return "\n".join(out)


def h_peel_body(bs, tw):
    """Interior (no edge mask) variant of h_loop_body with the warm-up peeled:
    the first PRO stream steps are straight-line code holding only the layer
    steps a stored output depends on (layer l starts at its index start(l):
    ~30% of the warm-up's layer steps drop out), every register is written
    before it is read (no zero fill), and the stream is shifted so the first
    stored column falls on a block boundary: the steady loop stores
    unconditionally."""
    L = len(bs)
    RX = lag(bs, L - 1)
    first_out = 2 * RX + L - 1
    PRO = (first_out + P - 1) // P * P
    shift = PRO - first_out
    Rs = [ring_size(2 * b + 1) for b in bs]
    regs = ["sv"] + [f"a{l}" for l in range(L + 1)] + [f"p{l}" for l in range(L)] + \
        [f"r{l}_{i}" for l in range(L) for i in range(Rs[l])]
    out = [f"    float2 {', '.join(regs)};"]
    for tau in range(shift, PRO):
        for l in reversed(range(L)):
            k = tau - shift - l
            if k < 0:
                continue
            if l == 0:
                out.append(f"    a0 = h2f2(in[{2 * k}]);")
            D = 2 * bs[l] + 1
            R = Rs[l]
            st = start(bs, l)
            if k < st:
                continue
            if k == st:
                out.append(f"    p{l} = a{l};")
                continue
            rd = f"r{l}_{(tau - l - D) % R}"
            wr = f"r{l}_{(tau - l) % R}"
            if k < st + D + 1:
                out.append(f"    {wr} = add2(a{l}, p{l}); p{l} = a{l};")
            else:
                out.append(f"    sv = add2(a{l}, p{l}); p{l} = a{l}; a{l + 1} = add2(sv, {rd}); {wr} = sv;")
    out.append("#pragma unroll 1")
    out.append(f"    for (int j = 0; j < {tw // P}; ++j) {{")
    out.append(f"        const unsigned *inj = in + {2 * (PRO - shift)} + {2 * P} * j;")
    out.append(f"        float2 *oj = out + {2 * P} * j;")
    for t in range(P):
        tau = PRO + t
        for l in reversed(range(L)):
            D = 2 * bs[l] + 1
            R = Rs[l]
            if l == 0:
                out.append(f"        a0 = h2f2(inj[{2 * t}]);")
            rd = f"r{l}_{(tau - l - D) % R}"
            wr = f"r{l}_{(tau - l) % R}"
            out.append(f"        sv = add2(a{l}, p{l}); p{l} = a{l}; a{l + 1} = add2(sv, {rd}); {wr} = sv;")
            if l == L - 1:
                out.append(f"        oj[{2 * t}] = a{L};")
    out.append("    }")
    # the tw % P columns after the last whole block (straight-line)
    nb = tw // P
    for t in range(tw % P):
        tau = PRO + t          # slot indices repeat with period P
        for l in reversed(range(L)):
            D = 2 * bs[l] + 1
            R = Rs[l]
            if l == 0:
                out.append(f"    a0 = h2f2(in[{2 * (PRO - shift + P * nb + t)}]);")
            rd = f"r{l}_{(tau - l - D) % R}"
            wr = f"r{l}_{(tau - l) % R}"
            out.append(f"    sv = add2(a{l}, p{l}); p{l} = a{l}; a{l + 1} = add2(sv, {rd}); {wr} = sv;")
            if l == L - 1:
                out.append(f"    out[{2 * (P * nb + t)}] = a{L};")
    return "\n".join(out)


def scalarize(text):
    """The float2 (channel pair per lane) H body as a one-channel-per-lane
    body: float state, plain adds, `in` a const __half * at element stride 4
    per pixel (RGBA), `out` a float * at stride 4 (kawase_sep_kernel<L, HS, true>)."""
    import re
    t = text
    t = re.sub(r"h2f2\((inj|in)\[(\d+)\]\)", lambda m: f"__half2float({m.group(1)}[{2 * int(m.group(2))}])", t)
    t = re.sub(r"add2\((\w+), (\w+)\)", r"(\1 + \2)", t)
    t = t.replace("make_float2(0.f, 0.f)", "0.f")
    t = re.sub(r"const unsigned \*inj = in \+ (\d+) \+ (\d+) \* j;",
               lambda m: f"const __half *inj = in + {2 * int(m.group(1))} + {2 * int(m.group(2))} * j;", t)
    t = re.sub(r"const unsigned \*inj = in \+ (\d+) \* j;",
               lambda m: f"const __half *inj = in + {2 * int(m.group(1))} * j;", t)
    t = re.sub(r"float2 \*oj = out \+ (\d+) \* j;", lambda m: f"float *oj = out + {2 * int(m.group(1))} * j;", t)
    t = re.sub(r"oj\[(\d+)\] =", lambda m: f"oj[{2 * int(m.group(1))}] =", t)
    t = t.replace("out[2 * oc]", "out[4 * oc]")
    t = re.sub(r"(\n\s*)out\[(\d+)\] =", lambda m: f"{m.group(1)}out[{2 * int(m.group(2))}] =", t)
    t = re.sub(r"\bfloat2 ", "float ", t)
    return t


def v_loop_state(bs):
    L = len(bs)
    Rs = [ring_size(2 * b + 1) for b in bs]
    return " ".join([f"float2 a{l};" for l in range(1, L)] + [f"float2 p{l};" for l in range(L)] +
                    [f"float2 r{l}_{i};" for l in range(L) for i in range(Rs[l])])


def v_loop_body(bs, lv=False):
    """One R-row iteration of the vertical passes as a loop over blocks of P
    rows (R % P == 0 and every ring size divides P: no rotation at the end).
    At local step t of block h layer l handles stream step 32 i + P h + t - l.
    Without MASK, a block whose P output rows all lie inside the segment's
    [y0, y1) (a per-block uniform test) stores unguarded."""
    assert R % P == 0
    L = len(bs)
    Rs = [ring_size(2 * b + 1) for b in bs]
    out = ["    float2 sv, a0;", "    const float2 z2 = make_float2(0.f, 0.f);",
           "    const long long rsb = rs * 2;      // output row pitch in bytes", "#pragma unroll 1",
           f"    for (int h = 0; h < {R // P}; ++h) {{",
           f"        const float2 *colh = col + h * {P} * HP2;",
           f"        const int th = {P} * h;",
           # a byte pointer stepped by the row pitch and kept opaque (the empty asm): without it
           # the compiler re-derives every row's address from the base (6 integer instructions per row)
           f"        char *orow = reinterpret_cast<char *>(outp) + (long long)(yout0 + th - {L - 1}) * rsb;"]

    def block(masked, guarded):
        for t in range(P):
            for l in reversed(range(L)):
                D = 2 * bs[l] + 1
                Rl = Rs[l]
                src = "a0" if l == 0 else f"S.a{l}"
                if l == 0 and lv:
                    # the last horizontal layer (b = bs[-1]) on load: columns x-b-1, x-b, x+b, x+b+1
                    # of the H warps' result, whose tile starts b + 1 columns left of the band
                    b = bs[-1]
                    out.append(f"        a0 = add2(add2(colh[{t} * HP2], colh[{t} * HP2 + 2]), "
                               f"add2(colh[{t} * HP2 + {2 * (2 * b + 1)}], colh[{t} * HP2 + {2 * (2 * b + 2)}]));")
                elif l == 0:
                    out.append(f"        a0 = colh[{t} * HP2];")
                dst = "a0" if l == L - 1 else f"S.a{l + 1}"
                rd = f"S.r{l}_{(t - l - D) % Rl}"
                wr = f"S.r{l}_{(t - l) % Rl}"
                out.append(f"        sv = add2({src}, S.p{l}); S.p{l} = {src}; {dst} = add2(sv, {rd}); {wr} = sv;")
                if masked:
                    out.append(f"        if (MASK && (unsigned)(yin0 + th + {t - l - lag(bs, l)}) >= (unsigned)H) {dst} = z2;")
                if l == L - 1:
                    if guarded:
                        out.append(f"        {{ const int yo = yout0 + th + {t - (L - 1)}; if (yo >= y0 && yo < y1) "
                                   f"st_h2(orow, mul2(a0, sc)); orow += rsb; asm volatile(\"\" : \"+l\"(orow)); }}")
                    else:
                        out.append(f"        st_h2(orow, mul2(a0, sc)); orow += rsb; asm volatile(\"\" : \"+l\"(orow));")

    out.append(f"        if (!MASK && yout0 + th - {L - 1} >= y0 && yout0 + th + {P - 1 - (L - 1)} < y1) {{")
    block(False, False)
    out.append("        } else {")
    block(True, True)
    out.append("        }")
    out.append("    }")
    return "\n".join(out)


def lv_members(bs):
    """LV: the H warps run the first L - 1 horizontal layers over the band plus
    b + 1 halo columns each side, and the V lanes apply the last horizontal
    layer when they load (4 loads and 3 adds instead of 1 load): the H warps
    are the critical path and the V warps wait on them."""
    L = len(bs)
    if L < 2:
        return "    static constexpr int kLvW = 0;"
    w = TW + 2 * (bs[-1] + 1)
    assert w % 2 == 0
    return f"""    static constexpr int kLvW = {w};          // H-result columns per band with the last layer left to V
    static constexpr int kLvReach = {lag(bs, L - 2)};       // reach of the first L - 1 layers
    template <bool EDGE>
    static __device__ __forceinline__ void h_half_lv(const unsigned *in, float2 *out, int xg0, int W) {{
{h_loop_body(bs[:-1], w // 2)}
    }}
    static __device__ __forceinline__ void h_half_lv_peel(const unsigned *in, float2 *out) {{
{h_peel_body(bs[:-1], w // 2)}
    }}
    template <bool MASK, int HP2>
    static __device__ __forceinline__ void v_lv(const float2 *col, State &S, int yin0, int H, int yout0, int y0,
                                                int y1, __half *outp, long long rs, float2 sc) {{
{v_loop_body(bs, lv=True)}
    }}"""


def emit():
    parts = ["// generated by gen_kawase.py -- do not edit", "template <int L> struct KwGen;"]
    for L in range(1, MAX_L + 1):
        bs = ladder(L)
        parts.append(f"""
template <> struct KwGen<{L}> {{
    static constexpr int kReach = {lag(bs, L - 1)};
    struct State {{ {v_loop_state(bs)} }};
    static __device__ __forceinline__ void zero(State &S) {{ memset(&S, 0, sizeof(S)); }}
    // a band's whole row / half / quarter (128 / 64 / 32 output columns):
    // the H work split over 1 / 2 / 4 times the lanes
    template <bool EDGE>
    static __device__ __forceinline__ void h(const unsigned *in, float2 *out, int xg0, int W) {{
{h_loop_body(bs, TW)}
    }}
    template <bool EDGE>
    static __device__ __forceinline__ void h_half(const unsigned *in, float2 *out, int xg0, int W) {{
{h_loop_body(bs, TW // 2)}
    }}
    template <bool EDGE>
    static __device__ __forceinline__ void h_quarter(const unsigned *in, float2 *out, int xg0, int W) {{
{h_loop_body(bs, TW // 4)}
    }}
    // interior rows with the warm-up peeled (no edge masks)
    static __device__ __forceinline__ void h_peel(const unsigned *in, float2 *out) {{
{h_peel_body(bs, TW)}
    }}
    static __device__ __forceinline__ void h_half_peel(const unsigned *in, float2 *out) {{
{h_peel_body(bs, TW // 2)}
    }}
    static __device__ __forceinline__ void h_quarter_peel(const unsigned *in, float2 *out) {{
{h_peel_body(bs, TW // 4)}
    }}
    // one channel per lane (scalar fp32 state): twice the H lanes at half the registers
    template <bool EDGE>
    static __device__ __forceinline__ void h_half_sc(const __half *in, float *out, int xg0, int W) {{
{scalarize(h_loop_body(bs, TW // 2))}
    }}
    static __device__ __forceinline__ void h_half_peel_sc(const __half *in, float *out) {{
{scalarize(h_peel_body(bs, TW // 2))}
    }}
{lv_members(bs)}
    // HP2 = H-result row pitch in float2
    template <bool MASK, int HP2>
    static __device__ __forceinline__ void v(const float2 *col, State &S, int yin0, int H, int yout0, int y0, int y1,
                                             __half *outp, long long rs, float2 sc) {{
{v_loop_body(bs)}
    }}
}};""")
    return "\n".join(parts) + "\n"


if __name__ == "__main__":
    text = emit()
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
