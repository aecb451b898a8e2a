"""Directive language (docs/directives.md): the host C++ parser vs the
reference's parse_directive/unparse (directive.hpp:522-554) — same spec,
same canonical text, same ParseErrorCode and byte offset on failures."""
import ctypes as C

import numpy as np
import pytest

from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E

FIELDS = [f for f, _ in abi.Spec._fields_ if f not in ("reserved0", "perfo_seed")]

VALID = [
    "memo(in:2:0.5f:4) level(warp) in(input[i*5:5:N]) out(output1[i])",
    "memo(out:3:5:1.5f) level(thread) out(output2[i])",
    "perfo(small:4)",
    "out(y[i]) level(team) memo(out:1:2:0.5)",
    "approx memo(out:1:2:0.5) level(block) out(y[i])",
    "memo(out:1:2:5) out(y[i])", "memo(out:1:2:inf) out(y[i])", "memo(out:1:2:INFINITY) out(y[i])",
    "memo(in:2:0.5) in(a[i],b[i*2+1:3]) out(y[i])",
    "memo(in:2:0.5) in(a[i]) in(b[i*2+1:3]) out(y[i])",
    "perfo(herded_large:8) level(warp)", "perfo(fini:20)", "perfo(ini:99)",
    "memo(in:8:1e-3:32) in(x[-3+i*4:7:M]) out(z[2])", "  memo ( out : 5 : 8 : 0.25 )  out ( y [ i - 2 ] )",
    "memo(out:2:3:1.0) out(y[i+0], z[3*i-1:N:K])", "memo(in:1:0) level(team) in(q[i]) out(r[i])",
]
MALFORMED = [
    "", "   ", "frobnicate(3)", "memo(out:1:2) out(y[i])", "memo(out:1:2:3:4) out(y[i])",
    "memo(in:x:0.5) in(a[i]) out(y[i])", "memo(out:1:2:zz) out(y[i])",
    "memo(out:1:2:3) perfo(small:4) out(y[i])", "level(warp) level(team) perfo(small:4)",
    "memo(inout:1:2) out(y[i])", "perfo(tiny:4)", "perfo(small:4) level(grid)",
    "memo(in:2:0.5) in(a[i*i:2]) out(y[i])", "memo(in:2:0.5) in(a[j]) out(y[i])",
    "perfo(ini:0)", "perfo(small:1)", "memo(in:0:0.5) in(a[i]) out(y[i])",
    "memo(in:2:0.5:4) out(y[i])", "memo(out:1:2:3)", "memo(out:1:2:0.5",
    "memo(out:1:2:-0.5) out(y[i])", "memo(out:1:2:nan) out(y[i])", "memo(out:1:2:+0.5) out(y[i])",
    "perfo(fini:100)", "memo(in:2:0.5) in(a[i:0]) out(y[i])", "memo(in:2:0.5) in(a[i:2:i]) out(y[i])",
    "memo(in:2:0.5) in(a[]) out(y[i])", "memo(in:2:0.5) in(a[i) out(y[i])", "perfo(small 4)",
    "memo(out:1:2:0.5) out(y[i]) junk", "approx", "1memo(out:1:2:3)", "perfo(small:-3)",
]


def _ours(text):
    spec = abi.Spec()
    code, off = C.c_int32(-9), C.c_int64(-9)
    buf = C.create_string_buffer(2048)
    rc = abi.lib().hpac_parse_directive(text.encode(), C.byref(spec), C.byref(code), C.byref(off), buf, 2048)
    return rc, spec, code.value, off.value, buf.value.decode()


def _ref(lib, text):
    spec = abi.Spec()
    code, off = C.c_int32(-9), C.c_int64(-9)
    buf = C.create_string_buffer(2048)
    rc = lib.ref_parse_directive(text.encode(), C.byref(spec), C.byref(code), C.byref(off), buf, 2048)
    return rc, spec, code.value, off.value, buf.value.decode()


def _same(a, b, text):
    assert a[0] == b[0], (text, a[4], b[4])
    if a[0] == abi.OK:
        for f in FIELDS:
            assert getattr(a[1], f) == getattr(b[1], f) or (f.endswith("threshold") and np.isnan(getattr(a[1], f))), (text, f)
        assert a[4] == b[4], text  # canonical text
    else:
        assert (a[2], a[3]) == (b[2], b[3]), (text, a[4], b[4])
        assert a[4] == b[4], text  # message


@pytest.mark.ref
@pytest.mark.parametrize("text", VALID + MALFORMED)
def test_matches_reference(ref_lib, text):
    _same(_ours(text), _ref(ref_lib, text), text)


@pytest.mark.ref
def test_fuzzed_mutations_match_reference(ref_lib):
    rng = np.random.default_rng(7)
    alphabet = list("memoperfinoutlvl():,[]*+-._ 0123456789iNxy") + ["memo(", "perfo(", "level(", "in(", "out(", "inf", "0.5f"]
    n = 0
    for _ in range(3000):
        base = VALID[rng.integers(len(VALID))]
        s = list(base)
        for _ in range(int(rng.integers(1, 4))):
            op = rng.integers(3)
            pos = int(rng.integers(0, len(s) + 1))
            if op == 0 and s:
                del s[min(pos, len(s) - 1)]
            elif op == 1:
                s.insert(pos, alphabet[rng.integers(len(alphabet))])
            elif s:
                s[min(pos, len(s) - 1)] = alphabet[rng.integers(len(alphabet))]
        text = "".join(s)
        if "random" in text:
            continue
        _same(_ours(text), _ref(ref_lib, text), text)
        n += 1
    assert n > 2500


@pytest.mark.parametrize("text", VALID)
def test_round_trip_idempotent(text):
    rc, spec, _, _, canon = _ours(text)
    assert rc == 0
    rc2, spec2, _, _, canon2 = _ours(canon)
    assert rc2 == 0 and canon2 == canon
    for f in FIELDS:
        assert getattr(spec, f) == getattr(spec2, f)


def test_known_codes():
    # test_directive.cpp "each malformed-input class yields its designated diagnostic"
    codes = {"": 0, "frobnicate(3)": 1, "memo(out:1:2) out(y[i])": 3, "memo(out:1:2:3:4) out(y[i])": 3,
             "memo(in:x:0.5) in(a[i]) out(y[i])": 4, "memo(out:1:2:3) perfo(small:4) out(y[i])": 5,
             "level(warp) level(team) perfo(small:4)": 5, "memo(inout:1:2) out(y[i])": 6,
             "perfo(tiny:4)": 7, "perfo(small:4) level(grid)": 8, "memo(in:2:0.5) in(a[j]) out(y[i])": 9,
             "perfo(ini:0)": 10, "memo(in:2:0.5:4) out(y[i])": 11, "memo(out:1:2:3)": 12,
             "memo(out:1:2:0.5": 2}
    for text, code in codes.items():
        with pytest.raises(E.DirectiveError) as ei:
            E.parse_directive(text)
        assert ei.value.code == code, text


def test_random_perforation_extension():
    spec, canon = E.parse_directive("perfo(random:30) level(warp)")
    assert spec.perfo_kind == abi.PERFO_RANDOM and spec.perfo_skip_percent == 30
    assert canon == "perfo(random:30) level(warp)"
    assert E.unparse(spec) == canon


def test_unparse_programmatic_specs():
    assert E.unparse(E.taf(5, 8, 0.5)) == "memo(out:5:8:0.5)"
    assert E.unparse(E.iact(4, 0.5, None, "team")) == "memo(in:4:0.5) level(team)"
    assert E.unparse(E.iact(2, float("inf"), 4)) == "memo(in:2:inf:4)"
    assert E.unparse(E.perfo("herded_small", 3, "warp")) == "perfo(herded_small:3) level(warp)"
