"""Bank-conflict analysis of the warp-engine buffer layout (tools/swizzle_check.py,
DESIGN.md §5 KB1): the shipped padding j + (j >> 4) costs 1.51x the ideal shared
wavefronts over all pass patterns (4-way on the LO = 4 pass of the split-tail
schedule); the XOR swizzle checked here is conflict-free and linear, but ptxas
turned its per-element address XORs into extra IMAD.MOV / IMAD.SHL on the
fmaheavy pipe and the kernel measured 2 % slower (profiles/r02/swizzle), so it
is not shipped.  These tests keep the analysis honest."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("swz", os.path.join(ROOT, "tools", "swizzle_check.py"))
S = importlib.util.module_from_spec(spec)
spec.loader.exec_module(S)


def test_swizzle_is_a_bijection_of_the_buffer():
    assert sorted(S.wswz(j) for j in range(1024)) == list(range(1024))
    # the values the C++ static_assert pins
    assert (S.wswz(16), S.wswz(32), S.wswz(64)) == (21, 42, 76)


def test_swizzle_is_linear_so_group_offsets_are_constants():
    for a in range(0, 1024, 7):
        for b in range(1024):
            if a & b == 0:
                assert S.wswz(a + b) == S.wswz(a) ^ S.wswz(b)


def test_every_pass_is_conflict_free():
    got, ideal = S.total(S.wswz)
    assert got == ideal
    got_pad, _ = S.total(S.pad)
    assert got_pad > ideal
