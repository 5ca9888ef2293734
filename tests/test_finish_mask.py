"""The FP32 strip engine's closed-form finish masks (dtw_f32.cuh) equal the
chained per-step updates they replace, for blocks of 8 and 16 steps, on
random and edge-case warps (pure bit arithmetic, checked on the CPU)."""
import random

import pytest

FULL = 0xFFFFFFFF


def chained(F, D, u0, BLK):
    """finmask |= D & ((finmask << 1) | (j0 + u > hi)), u = 0..BLK-1, with
    j0 + u > hi  <=>  u >= u0."""
    for u in range(BLK):
        c = 1 if u >= u0 else 0
        F |= D & (((F << 1) & FULL) | c)
    return F


def closed(F, D, u0, BLK):
    """dtw_f32.cuh: bounded propagation through D by doubling (1, 2, 4, ...
    up to a reach of BLK - 1), plus the lane-0 run."""
    G = ((F << 1) & FULL) & D
    P = D
    sh = 1
    while sh < BLK:
        G |= P & ((G << sh) & FULL)
        if 2 * sh < BLK:
            P &= (P << sh) & FULL
        sh *= 2
    u0 = max(0, u0)
    if u0 < BLK:
        inv = ~D & FULL
        run = 32 if inv == 0 else (inv & -inv).bit_length() - 1  # trailing ones of D
        k = min(run, BLK - u0)
        G |= FULL if k >= 32 else (1 << k) - 1
    return F | G


@pytest.mark.parametrize("BLK", [8, 16])
def test_closed_form_equals_chained_updates(BLK):
    rng = random.Random(2010_05371 + BLK)
    cases = 0
    for _ in range(60000):
        mode = rng.random()
        if mode < 0.3:  # runs of dead lanes, the common shape
            D = 0
            for _ in range(rng.randint(0, 4)):
                a = rng.randint(0, 31)
                b = rng.randint(a, min(31, a + rng.randint(0, 20)))
                D |= ((1 << (b - a + 1)) - 1) << a
        else:
            D = rng.getrandbits(32)
        F = rng.getrandbits(32) & rng.getrandbits(32) if rng.random() < 0.7 else 0
        u0 = rng.randint(-3, BLK + 4)
        assert closed(F, D, u0, BLK) == chained(F, D, u0, BLK), (hex(F), hex(D), u0)
        cases += 1
    for D in (0, FULL, 1, 0x7F, 0xFF, 0x80000000, 0xFFFF0000):
        for F in (0, 1, 0x80000000, FULL, 0x00F0F000):
            for u0 in range(-1, BLK + 2):
                assert closed(F, D, u0, BLK) == chained(F, D, u0, BLK)
    assert cases == 60000
