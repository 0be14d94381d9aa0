"""The reference-side binding without a GPU: install() swaps exactly the
reference's executor names (spmmlab.sim.run and the runner's imported
run), uninstall() restores them, and a call fails loudly (no CPU fallback)
when no CUDA device is visible."""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


@pytest.fixture()
def spmmlab_ref():
    if not (REF / "spmmlab").exists():
        pytest.skip("reference install baseline/_ref absent")
    sys.path.insert(0, str(REF))
    import spmmlab.runner  # noqa: F401
    import spmmlab.sim  # noqa: F401
    return sys.modules["spmmlab"]


def test_install_swaps_and_restores_the_executor(spmmlab_ref):
    import spmmlab.runner as R
    import spmmlab.sim as S
    from integration import spmmlab_b200 as I
    orig_sim, orig_runner = S.run, R.run
    I.install()
    try:
        assert S.run is I.run and R.run is I.run
        I.install()  # idempotent: the saved originals are not overwritten
    finally:
        I.uninstall()
    assert S.run is orig_sim and R.run is orig_runner


def test_no_cpu_fallback(spmmlab_ref):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import spmmlab.matrices as M
    import spmmlab.runner as R
    from integration import spmmlab_b200 as I
    a = M.random_csr(32, 32, 0.1, seed=1)
    b = M.random_dense(32, 8, seed=2)
    k = R.build_kernel(R.parse_point("row:1,col:1,r:1"), R.KernelConfig(n=8, p=256), a)
    with pytest.raises(RuntimeError, match="CUDA"):
        I.run(k, a, b)
