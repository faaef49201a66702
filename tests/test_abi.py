"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, its host-side Philox matches the Random123 known answers and
the oracle's independent Python Philox, and the schedule agrees with the
oracle's schedule.  No compute call is made (no device here)."""
import os
import re

import numpy as np
import pytest

from oracle import asyflexa_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1701_04900_b200 import build
    build.build()
    from paper_1701_04900_b200 import asyflexa
    return asyflexa


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "asyflexa.h")).read()
    declared = set(re.findall(r"ASY_API\s+[\w\s\*]+?\b(asy_\w+)\s*\(", hdr))
    assert len(declared) >= 12
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (asy_\w+)", out))
    assert declared <= exported, declared - exported


KAT = [  # Random123 kat_vectors, philox4x32_10
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(lib, ctr, key, want):
    assert lib.asy_philox4x32_10(ctr, key) == want
    assert O.philox4x32_10(ctr, key) == want


@pytest.mark.parametrize("nblocks", [1, 2, 7, 64, 625, 1000])
def test_schedule_matches_oracle_and_is_permutation(lib, nblocks):
    for seed in (0, 12345, 2 ** 40 + 7):
        for epoch in (0, 1, 5):
            order = O.random_epoch_order(seed, epoch, nblocks)
            assert sorted(order) == list(range(nblocks))
            got = [lib.asy_schedule_block(lib.ASY_SCHED_RANDOM, seed, nblocks, epoch * nblocks + i)
                   for i in range(nblocks)]
            assert got == order
    assert [lib.asy_schedule_block(lib.ASY_SCHED_CYCLIC, 3, nblocks, k) for k in range(2 * nblocks)] == \
        list(range(nblocks)) * 2


@pytest.mark.parametrize("sched", ["cyclic", "random"])
@pytest.mark.parametrize("nblocks", [1, 5, 64, 625])
def test_schedule_prev_is_previous_occurrence(lib, sched, nblocks):
    """asy_schedule_prev (the D4 guard of the dense kernel) against a brute-force scan
    of the oracle's schedule: the last earlier sequence that updated the same block."""
    sc = lib.ASY_SCHED_CYCLIC if sched == "cyclic" else lib.ASY_SCHED_RANDOM
    for seed in (0, 99):
        order = (O.cyclic_schedule(nblocks, 3) if sched == "cyclic"
                 else [b for e in range(3) for b in O.random_epoch_order(seed, e, nblocks)])
        last = {}
        for k, b in enumerate(order):
            assert lib.asy_schedule_prev(sc, seed, nblocks, k) == last.get(b, -1)
            last[b] = k


def test_random_epochs_differ(lib):
    a = O.random_epoch_order(1, 0, 500)
    b = O.random_epoch_order(1, 1, 500)
    c = O.random_epoch_order(2, 0, 500)
    assert a != b and a != c


def test_invalid_arguments_no_device(lib):
    with pytest.raises(lib.AsyError):
        lib.asy_schedule_block(7, 0, 10, 0)
    with pytest.raises(lib.AsyError):
        lib.asy_schedule_block(0, 0, 0, 0)
    # without a GPU asy_create must fail cleanly (error code, message), not crash
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        with pytest.raises(lib.AsyError) as ei:
            lib.asy_create(0)
        assert ei.value.code in (lib.ASY_ERR_CUDA, lib.ASY_ERR_UNSUPPORTED)
        assert lib.asy_last_error(None)
