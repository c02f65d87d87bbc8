"""CPU check of the generated Kawase H bodies (csrc/gen_kawase.py): the
emitted statements are translated to Python and run on one random row, then
compared with the direct chain of 1-D Kawase sums.  Run by tests/test_host.py."""
import re
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "paper_2512_04556_b200" / "csrc"))
import gen_kawase as g  # noqa: E402


def run_body(body, inp):
    lines, ind = [], 0
    for ln in body.split("\n"):
        s = ln.strip()
        m = re.match(r"float2? \*oj = out \+ (\d+) \* j;", s)
        if m:
            lines.append(" " * ind + f"oj = {m.group(1)}*j")
            continue
        if re.match(r"float2? [a-z]", s) or s.startswith("#pragma") or s.startswith("z2 ="):
            continue
        if s.startswith("for (int j"):
            n = int(re.search(r"j < (\d+)", s).group(1))
            lines.append(" " * ind + f"for j in range({n}):")
            ind += 4
            continue
        if s == "}":
            ind -= 4
            continue
        m = re.match(r"const (?:unsigned|__half) \*inj = in \+ (\d+) \+ (\d+) \* j;", s)
        if m:
            lines.append(" " * ind + f"inj = {m.group(1)} + {m.group(2)}*j")
            continue
        for st in s.split(";"):
            st = st.strip()
            if not st:
                continue
            st = re.sub(r"(?:h2f2|__half2float)\(inj\[(\d+)\]\)", r"IN[inj+\1]", st)
            st = re.sub(r"(?:h2f2|__half2float)\(in\[(\d+)\]\)", r"IN[\1]", st)
            st = re.sub(r"add2\((\w+), (\w+)\)", r"(\1+\2)", st)
            st = re.sub(r"oj\[(\d+)\] = (\w+)", r"OUT[oj+\1] = \2", st)
            st = re.sub(r"^out\[(\d+)\] = (\w+)", r"OUT[\1] = \2", st)
            lines.append(" " * ind + st)
    env = {"IN": inp, "OUT": {}}
    exec("\n".join(lines), env)
    return env["OUT"]


def run_loop_body(body, inp, xg0, W, edge):
    """h_loop_body's text as Python (EDGE, xg0, W bound at run time)."""
    lines, ind = [], 0
    for ln in body.split("\n"):
        s = ln.strip()
        if re.match(r"float2? [a-z]", s) or s.startswith("#pragma"):
            continue
        if s.startswith("for (int j"):
            n = int(re.search(r"j < (\d+)", s).group(1))
            lines.append(" " * ind + f"for j in range({n}):")
            ind += 4
            continue
        m = re.match(r"if \(EDGE && \((.*)\)\) \{", s)
        if m:
            lines.append(" " * ind + "if EDGE and (" + m.group(1).replace("||", "or") + "):")
            ind += 4
            continue
        if s == "} else {":
            lines.append(" " * (ind - 4) + "else:")
            continue
        if s == "}":
            ind -= 4
            continue
        m = re.match(r"const (?:unsigned|__half) \*inj = in \+ (\d+) \* j;", s)
        if m:
            lines.append(" " * ind + f"inj = {m.group(1)}*j")
            continue
        m = re.match(r"const int kj = (\d+) \* j;", s)
        if m:
            lines.append(" " * ind + f"kj = {m.group(1)}*j")
            continue
        m = re.match(r"if \(\(unsigned\)\((.*)\) >= \(unsigned\)W\) (\w+) = z2;", s)
        if m:
            lines.append(" " * ind + f"if not (0 <= ({m.group(1)}) < W): {m.group(2)} = 0.0")
            continue
        m = re.match(r"\{ const int oc = kj \+ (-?\d+); if \(\(unsigned\)oc < (\d+)u\) out\[(\d) \* oc\] = (\w+); \}", s)
        if m:
            lines.append(" " * ind + f"oc = kj + {m.group(1)}")
            lines.append(" " * ind + f"if 0 <= oc < {m.group(2)}: OUT[{m.group(3)}*oc] = {m.group(4)}")
            continue
        for st in s.split(";"):
            st = st.strip()
            if not st:
                continue
            st = st.replace("make_float2(0.f, 0.f)", "0.0").replace("0.f", "0.0")
            st = re.sub(r"(?:h2f2|__half2float)\(inj\[(\d+)\]\)", r"IN.get(inj+\1, 0.0)", st)
            st = re.sub(r"add2\((\w+), (\w+)\)", r"(\1+\2)", st)
            lines.append(" " * ind + st)
    env = {"IN": inp, "OUT": {}, "EDGE": edge, "xg0": xg0, "W": W}
    exec("\n".join(lines), env)
    return env["OUT"]


def check_loop(scalar=False):
    """Rolled bodies, interior and with the image edge anywhere in the band
    (zero padding re-applied after every layer: engine.py:106-115 per layer)."""
    for L in (1, 3, 6):
        for tw in (g.TW, g.TW // 2, 70):
            bs = g.ladder(L)
            RX = g.lag(bs, L - 1)
            W = 300
            img = np.random.default_rng(7 * L).random(W)
            ref = img.copy()
            for b in bs:
                ref = h4(ref, b)      # h4 zero-pads and returns the in-image positions only
            st = 4 if scalar else 2
            body = g.scalarize(g.h_loop_body(bs, tw)) if scalar else g.h_loop_body(bs, tw)
            for xs in (0, 64, W - tw - RX + 3, W - tw, W - tw + 17, W - 5):
                xg0 = xs - RX
                inp = {st * k: (img[xg0 + k] if 0 <= xg0 + k < W else 0.0) for k in range(tw + 2 * RX + 64)}
                edge = xs - RX < 0 or xs + tw + RX > W
                out = run_loop_body(body, inp, xg0, W, edge)
                assert sorted(out) == [st * i for i in range(tw)], (L, tw, xs)
                for i in range(tw):
                    if xs + i < W:
                        assert abs(out[st * i] - ref[xs + i]) <= 1e-12 * abs(ref[xs + i]), (L, tw, xs, i)


def h4(v, b):
    pad = np.zeros(len(v) + 2 * (b + 1))
    pad[b + 1:b + 1 + len(v)] = v
    i = np.arange(len(v)) + b + 1
    return pad[i - b - 1] + pad[i - b] + pad[i + b] + pad[i + b + 1]


def check_peel(scalar=False):
    st = 4 if scalar else 2      # index stride per pixel of `in` and `out`
    for L in range(1, g.MAX_L + 1):
        for tw in (g.TW, g.TW // 2, g.TW // 4, 70):
            bs = g.ladder(L)
            RX = g.lag(bs, L - 1)
            x = np.random.default_rng(L).random(tw + 2 * RX + 40)
            body = g.h_peel_body(bs, tw)
            out = run_body(g.scalarize(body) if scalar else body, {st * k: x[k] for k in range(len(x))})
            v = x.copy()
            for b in bs:
                v = h4(v, b)
            assert sorted(out) == [st * i for i in range(tw)], (L, tw)
            got = np.array([out[st * i] for i in range(tw)])
            assert np.allclose(got, v[RX:RX + tw], rtol=1e-13, atol=0), (L, tw)


if __name__ == "__main__":
    for sc in (False, True):
        check_peel(sc)
        check_loop(sc)
    print("peel bodies ok")
