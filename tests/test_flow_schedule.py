"""The ticket schedule of the dataflow polymul kernel (k_flow, ntt_large.cuh),
mirrored in Python: every (phase, unit, tile) is issued exactly once, and every
tile's dependencies (all tiles of the previous phase of its unit) carry smaller
tickets -- the property the kernel's deadlock freedom rests on (a dependency is
always held by a CTA that is already running)."""
import pytest

LAG = 7     # kFlowLag
T = 16      # tiles per phase at N = 2^16 (R / kColTile = R / RPC)


def schedule(units):
    rounds = units + 2 * LAG
    out = {}
    for t in range(3 * T * rounds):
        r, slot = divmod(t, 3 * T)
        phase, tile = divmod(slot, T)
        unit = r - phase * LAG
        if 0 <= unit < units:
            assert (phase, unit, tile) not in out
            out[(phase, unit, tile)] = t
    return out


@pytest.mark.parametrize("units", [1, 2, 7, 45, 480])
def test_every_tile_once_and_dependencies_earlier(units):
    s = schedule(units)
    assert len(s) == 3 * T * units
    for (phase, unit, tile), t in s.items():
        if phase:
            assert all(s[(phase - 1, unit, k)] < t for k in range(T))


def test_header_constants_match():
    import os
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_2410_05934_b200", "csrc", "ntt_large.cuh")).read()
    assert "constexpr int kFlowLag = 7;" in src
