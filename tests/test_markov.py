"""Markovian engine (paper_2604_22092_b200.markov, csrc/fs_markov.cu) against
the reference's own markov_step / run_markov (tests/golden/make_markov_golden.py):
per-step clock, tau and counts, final states / rates / influence, and the
run_markov record — bit for bit.  Also the reference's unit tests
(T/test_markov.py) that apply to the device engine."""

import json

import numpy as np
import pytest

import paper_2604_22092_b200 as fs
from paper_2604_22092_b200.models import Holding, ModelSpec
from tests._cases import GOLDEN

MARKOV = json.loads((GOLDEN / "markov.json").read_text())
SIS = fs.sis_model(0.25, 0.15)
SIR = fs.sir_model(0.25, 0.15)


def seir_exp():
    return ModelSpec(name="seir-exp", compartments=("S", "E", "I", "R"), beta=0.25, edge_from=0, edge_to=1,
                     nodal={1: (2, Holding.exponential(0.2)), 2: (3, Holding.exponential(1.0 / 7.5))}, infectious=2)


MODELS = {"sir": lambda: SIR, "sis": lambda: SIS, "seir_exp": seir_exp}


def golden():
    with np.load(GOLDEN / "markov.npz") as z:
        return {k: z[k] for k in z.files}


def case(name):
    meta = MARKOV[name]
    gs = meta["graph"]
    g = getattr(fs, gs[0])(*gs[1:3], seed=gs[3])
    return meta, g, MODELS[meta["model"]](), fs.MarkovConfig(**meta["cfg"])


def test_requires_exponential_and_constant():
    g = fs.gen_erdos_renyi(50, 4.0, seed=3)
    with pytest.raises(ValueError):
        fs.init_markov_state(g, fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0), np.array([0]))


def test_config_validation():
    with pytest.raises(ValueError):
        fs.MarkovConfig(p_max=1.5)
    with pytest.raises(ValueError):
        fs.MarkovConfig(theta=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(MARKOV))
def test_markov_steps_bit_exact(name):
    from paper_2604_22092_b200.renewal import _pick_seed_nodes

    ref = golden()
    meta, g, m, cfg = case(name)
    picked = _pick_seed_nodes(g.num_nodes, meta["seed"], meta["seed_count"], fs._device.device()).cpu().numpy()
    st = fs.init_markov_state(g, m, picked)
    clocks, taus, counts = [], [], []
    for _ in range(meta["steps"]):
        _, tau = fs.markov_step(st, g, m, cfg, meta["seed"])
        clocks.append(st.clock)
        taus.append(tau)
        counts.append(st.counts)
    assert np.array_equal(np.array(counts), ref[f"{name}__counts"])
    assert np.array_equal(np.array(taus), ref[f"{name}__tau"])
    assert np.array_equal(np.array(clocks), ref[f"{name}__clock"])
    assert np.array_equal(st.states, ref[f"{name}__states"])
    assert np.array_equal(st.rates, ref[f"{name}__rates"])
    assert np.array_equal(st.influence, ref[f"{name}__influence"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(MARKOV))
def test_run_markov_record_bit_exact(name):
    ref = golden()
    meta, g, m, cfg = case(name)
    rec = fs.run_markov(g, m, cfg, meta["seed"], meta["t_final"], seed_count=meta["seed_count"])
    assert rec.summary["step_count"] == int(ref[f"{name}__record_steps"])
    assert np.array_equal(rec.fractions, ref[f"{name}__record"])


@pytest.mark.gpu
def test_influence_matches_brute_force():
    g = fs.gen_erdos_renyi(100, 8.0, seed=2)
    states = np.random.default_rng(0).integers(0, 2, 100).astype(np.int32)
    got = fs.influence_gather(g, states, SIS)
    want = np.array([sum(float(states[c] == 1) for c in g.col_indices[g.row_offsets[i]:g.row_offsets[i + 1]])
                     for i in range(100)])
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_all_terminal_step_is_max_tau():
    # T/test_markov.py:70-80
    g = fs.gen_erdos_renyi(50, 4.0, seed=4)
    st = fs.init_markov_state(g, SIR, np.array([], dtype=np.int64))
    st.states[:] = 2
    st.counts = np.array([0, 0, 50], dtype=np.int64)
    _, tau = fs.markov_step(st, g, SIR, fs.MarkovConfig(), seed=1)
    assert tau == fs.MarkovConfig().tau_max
    assert np.array_equal(st.counts, [0, 0, 50])
