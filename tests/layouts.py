"""Rank layouts of the P > 1 GPU tests.

("gpus", P): P ranks on GPUs 0..P-1 (ks_create); skipped on a box with fewer GPUs.
("shared", P): P ranks all on GPU 0 (ks_create_on with a repeated device): the P > 1
schedule -- row-block partition, allgathers of r / p / v ingredients, rank-ordered
scalar sums, x gather -- through host-driven peer-copy collectives (no NCCL, no fused
exchange: kernels that wait on each other are never launched separately on one GPU,
B200_PROFILING.md) -- except as ONE cooperative launch over all ranks' CTAs: CG /
BiCGSTAB with x0 = 0 run the fused persistent / tiny kernels of all ranks that way.
It runs on any GPU box, so rows A4 / B2 (host-collective and fused) and the fused
exchange of NEXT-1 are checked against the oracle even where only one GPU exists;
NVLink itself and the multi-process path need the ("gpus", P) layouts.
"""
import pytest

PS_GPUS = (2, 4, 8)
PS_SHARED = (2, 4)


def ngpu():
    import torch
    return torch.cuda.device_count()


def layouts(gpus=PS_GPUS, shared=PS_SHARED):
    return ([pytest.param(("gpus", P), id=f"gpus{P}") for P in gpus] +
            [pytest.param(("shared", P), id=f"shared{P}") for P in shared])


def need(lay):
    """Skips when the box cannot host the layout; returns P."""
    mode, P = lay
    if ngpu() < 1:
        pytest.skip("needs a GPU")
    if mode == "gpus" and ngpu() < P:
        pytest.skip(f"needs {P} GPUs")
    return P


def context(n, lay, **kw):
    import paper_1511_07174_b200 as ks
    mode, P = lay
    if mode == "gpus":
        return ks.Context(n, ngpus=P, **kw)
    return ks.Context(n, devices=[0] * P, **kw)
