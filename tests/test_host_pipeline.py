"""conv_run_host's chunk plan (api.cpp compute_host_chunks), on a described
B200 (offline plans, no GPU): the image chunks are chosen by simulating the
upload / compute / download pipeline with the selector's model time of every
chunk's sub-problem (Alg. 1's evaluate-every-candidate
applied to the pipeline).  The GPU side (the chunks really pipeline and stay
bit-identical to conv_run) is tests/test_parity.py::test_run_host_*."""
import pytest

from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS

PATHS = ["fp32_simt", "fp32_tc", "tf32", "bf16"]
H2D, D2H = 55.2e9, 56.9e9          # the measured solo link rates (profiles/r02b/e2e/)


def _host(sh, path):
    return conv.ConvPlan(*sh.as_tuple(), path=path, offline_device=conv.B200).describe()["host_pipeline"]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["tiny", "r2", "pw", "det", "batched"])
def test_chunks_partition_the_batch(name, path):
    sh = CONFIGS[name]
    hp = _host(sh, path)
    ch = hp["chunks"]
    assert 1 <= len(ch) <= 32 and all(c >= 1 for c in ch) and sum(ch) == sh.N
    # the modeled pipeline is never shorter than the uploads plus the downloads at the solo rates
    # of the link minus their overlap: at least the longer of the two
    bi = 4 * sh.N * sh.C * sh.Hin * sh.Win
    bo = 4 * sh.N * sh.K * sh.H * sh.W
    assert hp["model_us"] >= max(bi / H2D, bo / D2H) * 1e6


@pytest.mark.parametrize("path", PATHS)
def test_batched_layer_is_pipelined(path):
    """67 MB in / 51 MB out: one chunk would serialise upload, compute and
    download; the plan pipelines them (several chunks) and models a time well
    under the serial sum."""
    sh = CONFIGS["batched"]
    d = conv.ConvPlan(*sh.as_tuple(), path=path, offline_device=conv.B200).describe()
    hp = d["host_pipeline"]
    assert len(hp["chunks"]) >= 4
    bi = 4 * sh.N * sh.C * sh.Hin * sh.Win
    bo = 4 * sh.N * sh.K * sh.H * sh.W
    assert hp["model_us"] < 0.85 * (bi / H2D + d["model"]["model_us"] * 1e-6 + bo / D2H) * 1e6


def test_single_image_layers_are_one_chunk():
    for name in ["tiny", "r2", "pw", "det"]:
        assert _host(CONFIGS[name], "fp32_simt")["chunks"] == [1]
