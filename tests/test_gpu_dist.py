"""GPU, >= 2 devices: one rank per GPU (torchrun), both collective paths, vs
the oracle (tools/dist_check.py). Skipped on a single-GPU box."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(nproc, *args, port=29577, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "dist_check.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=None if env is None else {**os.environ, **env})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PASS" in r.stdout


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync", ["p2p", "p2p-pull", "nccl"])
def test_two_ranks_bit_exact_vs_oracle(sync):
    _run(2, "--sync", sync, "--steps", "12")


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("holder_sum", ["0", "1"])
def test_two_ranks_push_reduce_holder_sum_switch(holder_sum):
    # the holder-sum exchange is the default from n = 4; force both ways at n = 2
    _run(2, "--sync", "p2p", "--steps", "12", port=29585, env={"EXD_HOLDER_SUM": holder_sum})


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_two_ranks_push_reduce_index_layouts():
    # the stream kernel pushes its indices packed per tile on large vectors and
    # as per-warp runs at the chunk's position on small ones; force the other way
    _run(2, "--sync", "p2p", "--steps", "10", port=29615, env={"EXD_TILE_PACK": "1"})
    _run(2, "--sync", "p2p", "--n_g", "20000003", "--steps", "5", "--skew", "0", port=29616,
         env={"EXD_TILE_PACK": "0"})


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_two_ranks_push_reduce_f64_vs_oracle():
    _run(2, "--sync", "p2p", "--dtype", "f64", "--steps", "8", port=29581)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync", ["p2p", "p2p-pull"])
def test_two_ranks_sparse_selection(sync):
    # k = 40 over 400k elements: partitions that select nothing, one-entry chunks
    _run(2, "--sync", sync, "--n_g", "400001", "--density", "0.0001", "--steps", "16", port=29582)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_two_ranks_density_cap():
    _run(2, "--sync", "p2p", "--cap", "0.01", "--steps", "10", port=29578)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync", ["p2p", "nccl"])
def test_replica_divergence_detected_across_gpus(sync):
    _run(2, "--sync", sync, "--inject", "1", port=29579)


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("sync", ["p2p", "p2p-pull"])
def test_four_ranks_p2p_rank_order_sum_is_bit_exact(sync):
    _run(4, "--sync", sync, "--steps", "12", port=29580)


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs")
def test_four_ranks_push_reduce_dense_and_sparse():
    _run(4, "--sync", "p2p", "--density", "0.1", "--steps", "8", port=29583)
    _run(4, "--sync", "p2p", "--n_g", "400001", "--density", "0.0002", "--steps", "8", port=29584)


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs")
def test_four_ranks_push_reduce_all_push():
    _run(4, "--sync", "p2p", "--steps", "12", port=29586, env={"EXD_HOLDER_SUM": "0"})
    _run(4, "--sync", "p2p", "--dtype", "f64", "--steps", "6", port=29587)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync", ["nccl", "p2p"])
def test_dead_peer_fails_the_step_instead_of_hanging(sync):
    # NCCL path: async-error / timeout polling (EXD_NCCL_TIMEOUT_S); peer-memory
    # path: the kernels' 20 s poll limit. Then the engine refuses further steps.
    _run(2, "--sync", sync, "--kill-peer", "1", port=29588 if sync == "nccl" else 29589,
         env={"EXD_NCCL_TIMEOUT_S": "5"})


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync", ["p2p", "p2p-pull"])
def test_two_ranks_large_vector_published_range_counts(sync):
    # n_g > 3072 tiles: the exchange / finish kernels take their bases from the
    # blocks' published range words instead of summing every earlier tile
    _run(2, "--sync", sync, "--n_g", "20000003", "--steps", "6", "--skew", "0",
         port=29590 if sync == "p2p" else 29591)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("holder_sum", ["0", "1"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_two_ranks_two_pass_exchange(holder_sum, dtype):
    # the two-pass exchange loop (chosen by size at large k'), forced on
    _run(2, "--sync", "p2p", "--dtype", dtype, "--steps", "10", "--density", "0.05",
         port=29592 + 2 * (dtype == "f64") + int(holder_sum),
         env={"EXD_TWO_PASS": "1", "EXD_HOLDER_SUM": holder_sum})


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs")
def test_four_ranks_two_pass_exchange_holder_sum():
    _run(4, "--sync", "p2p", "--steps", "10", "--density", "0.05", port=29596,
         env={"EXD_TWO_PASS": "1"})
    _run(4, "--sync", "p2p", "--n_g", "20000003", "--steps", "5", "--skew", "0", port=29597)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("holder_sum", ["0", "1"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_two_ranks_bounded_inbox_spills_to_pull(holder_sum, dtype):
    # contribution slots for 3000 union positions only (EXD_PUSH_CAP): the rest
    # of every step's union goes through the sources' spill buffers and flags
    _run(2, "--sync", "p2p", "--dtype", dtype, "--steps", "10",
         port=29600 + 2 * (dtype == "f64") + int(holder_sum),
         env={"EXD_PUSH_CAP": "3000", "EXD_HOLDER_SUM": holder_sum})


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs")
def test_four_ranks_bounded_inbox_spills_to_pull():
    _run(4, "--sync", "p2p", "--steps", "10", port=29604, env={"EXD_PUSH_CAP": "3000"})
    _run(4, "--sync", "p2p", "--steps", "6", "--density", "0.1", port=29605,
         env={"EXD_PUSH_CAP": "100000", "EXD_HOLDER_SUM": "0"})


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("kind", ["topk", "cltk", "hardthreshold"])
def test_two_ranks_baseline_sparsifiers_over_nccl(kind):
    # one rank per GPU: counts and padded lists all-gathered over NCCL, the
    # deduplicating union on every rank, NCCL sum (exact at n = 2)
    _run(2, "--sparsifier", kind, "--steps", "8", port=29610 + ["topk", "cltk", "hardthreshold"].index(kind))


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs")
def test_four_ranks_baseline_sparsifiers_over_nccl():
    _run(4, "--sparsifier", "topk", "--steps", "6", port=29613)
    _run(4, "--sparsifier", "cltk", "--steps", "6", "--dtype", "f64", port=29614)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("env", ["EXD_TILE_PACK=1", "EXD_HOLDER_SUM=1", "EXD_PUSH_CAP=5000"])
def test_protocol_switches_must_agree_across_ranks(env):
    # the peers' kernels read each other's inbox layout: a switch set on one
    # rank only fails engine creation everywhere instead of corrupting the sum
    _run(2, "--sync", "p2p", "--mismatch-env", env,
         port=29620 + ["EXD_TILE_PACK=1", "EXD_HOLDER_SUM=1", "EXD_PUSH_CAP=5000"].index(env))
