"""CPU checks of the C-ABI library: it loads without a GPU, exports every
symbol include/mdr_sm100.h declares, and fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_2605_05208_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mdr_sm100.h")).read()
    return sorted(set(re.findall(r"\b(mdr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_exactly_the_bound_symbols():
    assert _declared() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(L, name), name


def test_no_gpu_means_loud_failure():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    assert _lib.device_count() == 0
    import random
    import paper_2605_05208_b200 as P
    from paper_2605_05208_b200 import workload as W
    inst = W.make_instance(random.Random(1), "mdvrp", n_customers=5)
    consts = P.ScalingConstants.from_instance(inst)
    with pytest.raises(RuntimeError):
        P.SolutionCache(W.random_solution(random.Random(2), inst), inst, consts)


def test_sm100a_code_is_in_the_library():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_native_shuffle_stream_equals_cpython_shuffle():
    """mdr_shuffle_stream reproduces random.Random.shuffle bit for bit (no GPU needed)."""
    import random
    from paper_2605_05208_b200.localsearch import _advance, draw_permutations
    for seed in (0, 1, 7, 12345, 2 ** 40 + 3):
        for ops in ([0, 1, 2, 4, 5], [0, 1, 2, 3, 4, 5], [3], list(range(20))):
            rng = random.Random(seed)
            rng.random()  # arbitrary prior consumption
            want_rng = random.Random()
            want_rng.setstate(rng.getstate())
            want = []
            for _ in range(700):  # crosses several MT19937 regenerations
                o = list(ops)
                want_rng.shuffle(o)
                want.append(o)
            got = draw_permutations(rng, ops, 700)
            assert got.tolist() == want
            _advance(rng, ops, 700)
            assert rng.getstate() == want_rng.getstate()
            assert rng.random() == want_rng.random()
