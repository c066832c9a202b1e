"""End-to-end parity at the BASELINE shapes: CUDA engine (C-ABI) vs the CPU oracle.

The c1 parity of tests/test_gpu_parity.py runs shapes that avoid the kernels the
large configs live on.  These cases run them:

* ``opt-125m`` (BASELINE.json configs[1] shape: OPT-125m x4, prompt 256 + response
  256) at batch 4 on one GPU.  S = 512 takes the fused tcgen05 attention forward
  (``attn_fwd_kernel``, T % 128 == 0, T <= 512) in prefill, the four Forwards and
  TrainFB; B*S = 2048 rows put the FFN / LM-head GEMMs on the CTA-pair kernel
  (``gemm_pair_kernel``, >= 74 256x256 tiles) and the Forward-stage logprobs on its
  log-sum-exp epilogue (logits never stored); decode runs the cluster split-K
  decode GEMMs and the bulk-copy ring attention; backward runs the split-K
  weight gradients.
* ``llama-mid`` (LLaMA family, d 1024, 4 layers, head_dim 128 = the 7B's, SwiGLU,
  rotary, untied head, V 32000), prompt 256 + response 256, batch 2.

The oracle is run teacher-forced on the GPU's own sequences, so every downstream
quantity is compared on identical inputs.  Tolerances (stated here, calibrated
from the observed spread at these depths):
  * greedy tokens: bit-exact wherever the oracle's top-2 margin > 5e-2;
  * logprobs / values / score / rewards: abs 5e-2 (12 bf16-rounded layers + V = 50272);
    LLaMA-mid logprobs abs 1e-1 (measured on B200: max 7.2e-2 in 1 of 512 entries, whose
    logprob is -13: a bf16 flip of the final RMSNorm output moves a far-from-top logit
    most), and for every quantity the MEAN abs error <= 1e-2 (LLaMA-mid logprobs 2e-2;
    measured 1.4e-2);
  * advantages / returns: abs 1e-1 (sums of up to R such terms, gamma*lam = 0.95);
  * losses: rel 3e-2;  gradients: per-tensor rel-L2 <= 5e-2;
  * updated fp32 masters: |delta| <= 2*lr + 1e-7, <= 1 % sign-flipped updates.
The persistent decode loop (OPT only) is checked against the oracle's greedy
predictions too, not only against the graph path.
"""
import numpy as np
import pytest

from paper_2312_11819_b200.capi import make_config, named_slices
from tests import oracle_lib

pytestmark = pytest.mark.gpu

CASES = {"opt-125m": (4, 256, 256), "llama-mid": (2, 256, 256)}
MARGIN = 5e-2


@pytest.fixture(scope="module", params=sorted(CASES))
def run(request):
    from paper_2312_11819_b200.engine import Engine
    B, P, R = CASES[request.param]
    cfg = make_config(request.param, request.param, B, P, R)
    eng = Engine(cfg)
    rep = eng.step()
    out = {k: eng.read(k) for k in ("tokens", "logp_old", "logp_ref", "values", "score", "rewards", "advantages",
                                    "returns", "logp_new", "values_new", "actor_grad", "critic_grad",
                                    "actor_master", "critic_master")}
    ora = oracle_lib.ppo_step(cfg, tokens_in=out["tokens"])
    return request.param, cfg, rep, out, ora


def test_greedy_tokens(run):
    _, cfg, _, out, ora = run
    P = cfg.prompt_len
    np.testing.assert_array_equal(out["tokens"][:, :P], ora["tokens"][:, :P])
    m = ora["greedy_margin"] > MARGIN
    assert m.mean() > 0.8, m.mean()
    np.testing.assert_array_equal(out["tokens"][:, P:][m], ora["greedy_pred"][m])


@pytest.mark.parametrize("key,atol", [("logp_old", 5e-2), ("logp_ref", 5e-2), ("values", 5e-2), ("score", 5e-2),
                                      ("rewards", 5e-2), ("advantages", 1e-1), ("returns", 1e-1),
                                      ("logp_new", 5e-2), ("values_new", 5e-2)])
def test_experience_and_training_forward(run, key, atol):
    name, _, _, out, ora, = run
    mean_tol = 1e-2
    if name == "llama-mid" and key.startswith("logp"):
        atol, mean_tol = 1e-1, 2e-2  # measured: max 7.2e-2, mean 1.4e-2 (logprobs near -10, V = 32000)
    err = np.abs(out[key] - ora[key])
    print(f"{name} {key}: max abs err {err.max():.3e}, mean {err.mean():.3e}")
    assert err.mean() <= mean_tol, err.mean()
    np.testing.assert_allclose(out[key], ora[key], atol=atol, rtol=1e-3)


def test_losses(run):
    _, _, rep, _, ora = run
    np.testing.assert_allclose([rep["actor_loss"], rep["critic_loss"]], [ora["actor_loss"], ora["critic_loss"]],
                               rtol=3e-2)


@pytest.mark.parametrize("tag", ["actor", "critic"])
def test_gradients(run, tag):
    name, cfg, _, out, ora = run
    arch = cfg.actor if tag == "actor" else cfg.critic
    g, go = out[f"{tag}_grad"], ora[f"{tag}_grad"]
    worst = 0.0
    for tname, off, n in named_slices(arch):
        a, b = g[off:off + n].astype(np.float64), go[off:off + n].astype(np.float64)
        err = np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12)
        worst = max(worst, err)
        assert err <= 5e-2, (tname, err)
    print(f"{name} {tag}: worst per-tensor grad rel-L2 {worst:.3e}")


@pytest.mark.parametrize("tag,lr", [("actor", 1e-5), ("critic", 5e-6)])
def test_updated_weights(run, tag, lr):
    _, _, _, out, ora = run
    mine, ref = out[f"{tag}_master"], ora[f"{tag}_master"]
    assert np.abs(mine - ref).max() <= 2 * lr + 1e-7
    moved = np.abs(ora[f"{tag}_grad"]) > 1e-6
    flips = np.mean(np.abs(mine[moved] - ref[moved]) > lr)
    assert flips <= 0.01, flips


def test_teacher_forced_decode_matches_oracle(run):
    from paper_2312_11819_b200.engine import Engine
    _, cfg, _, out, ora = run
    pred, margin = Engine(cfg).greedy_check(out["tokens"])
    m = ora["greedy_margin"] > MARGIN
    np.testing.assert_array_equal(pred[m], ora["greedy_pred"][m])
    np.testing.assert_allclose(margin, ora["greedy_margin"], atol=1e-1)


def test_persistent_decode_loop_matches_oracle(run):
    """rlhf_decode_loop (all decode steps in one cooperative kernel) against the oracle."""
    from paper_2312_11819_b200.engine import Engine
    name, cfg, _, out, ora = run
    if name != "opt-125m":
        pytest.skip("the persistent decode loop implements the OPT family")
    pred, margin = Engine(cfg, cuda_graph=3).greedy_check(out["tokens"])
    m = ora["greedy_margin"] > MARGIN
    np.testing.assert_array_equal(pred[m], ora["greedy_pred"][m])
    np.testing.assert_allclose(margin, ora["greedy_margin"], atol=1e-1)
