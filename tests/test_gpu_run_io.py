"""The GPU training driver and run directories
against the reference's own EM loop (em.cpp run, annealing, weight noise,
tolerance stop; oracle/_ref ``ref_train``) and run-directory layout
(run_io.cpp: free_energy.csv, checkpoint cadence, final arrays, manifest).
"""
import csv
import json

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rio():
    import paper_1908_06843_b200 as P

    assert P._native.lib().prsp_bsc_gpu_device_count() > 0, "no CUDA device: the sm_100a path cannot run"
    from paper_1908_06843_b200 import run_io

    return run_io


def bars(port, size=4, n=160, seed=3):
    y, _ = port.make_bars(size, n, seed=seed)
    return y


@pytest.mark.parametrize("model,values,h,hp,g", [
    ("bsc", None, 8, 6, 3),
    ("tsc", None, 8, 5, 3),
    ("dsc", [-1.0, 0.0, 1.0, 2.0], 8, 5, 2),
    ("mca", None, 8, 6, 3),
    ("mmca", None, 8, 5, 3),
])
def test_train_matches_reference_loop(rio, port, ref, model, values, h, hp, g):
    y = bars(port)
    cfg = rio.TrainConfig(model=model, latents=h, hprime=hp, gamma=g, values=values, iterations=4, seed=7)
    r = rio.train(cfg, y)
    trace, w, pi, s2, probs = ref.train(model, y, h, hp, g, 4, 7, values=values)
    assert len(r.free_energy) == len(trace) == 4
    assert rel(r.free_energy, trace) < 1e-6, (r.free_energy, trace)
    assert rel(r.params["W"], w) < 1e-6
    assert abs(r.params["sigma2"][0, 0] - s2) <= 1e-6 * s2
    if model == "dsc":
        assert np.max(np.abs(r.params["probs"][0] - probs) / probs) < 1e-6
        assert np.array_equal(r.params["values"][0], values)
    else:
        assert abs(r.params["pi"][0, 0] - pi) <= 1e-6 * pi


def test_annealing_noise_and_tolerance(rio, port, ref):
    y = bars(port, seed=5)
    sched = dict(temperature=[(0.0, 3.0), (0.5, 1.0)], w_noise=[(0.0, 0.2), (0.5, 0.0)])
    r = rio.train(rio.TrainConfig(model="bsc", latents=8, hprime=6, gamma=3, iterations=6, seed=11, **sched), y)
    trace, w, pi, s2, _ = ref.train("bsc", y, 8, 6, 3, 6, 11, **sched)
    assert rel(r.free_energy, trace) < 1e-6 and rel(r.params["W"], w) < 1e-6
    # tolerance: stops at the same iteration as the reference (em.cpp:67-72)
    r = rio.train(rio.TrainConfig(model="bsc", latents=8, hprime=6, gamma=3, iterations=60, seed=11, tolerance=1e-4),
                  y)
    trace, *_ = ref.train("bsc", y, 8, 6, 3, 60, 11, tol=1e-4)
    assert len(trace) < 60 and len(r.free_energy) == len(trace)


def test_run_directory_and_reload(rio, port, tmp_path):
    import paper_1908_06843_b200 as P

    y = bars(port, seed=9)
    data = tmp_path / "data.prsp"
    rio.save_array(data, y)
    out = tmp_path / "run"
    cfg = rio.TrainConfig(model="tsc", latents=8, hprime=5, gamma=3, iterations=3, seed=2, workers=4, shards=4)
    r = rio.train(cfg, rio.load_dataset(data), data_file=str(data), out_dir=str(out))
    rows = list(csv.reader(open(out / "free_energy.csv")))
    assert rows[0] == ["iteration", "free_energy", "seconds"] and len(rows) == 4
    assert [float(x[1]) for x in rows[1:]] == list(r.free_energy)
    for prefix in ["checkpoint", "final"]:
        for name in ["W", "sigma2", "pi"]:
            assert (out / f"{prefix}_{name}.prsp").exists()
    assert np.array_equal(rio.load_array(out / "final_W.prsp"), r.params["W"])
    m = json.load(open(out / "manifest.json"))
    assert m["format"] == "prsp-manifest-1" and m["model"] == "tsc" and m["dim"] == y.shape[1]
    assert m["hprime"] == 5 and m["gamma"] == 3 and m["iterations"] == 3 and m["workers"] == 4
    assert m["data"]["sha256"] == rio.sha256_file(data) and m["data"]["rows"] == y.shape[0]
    assert m["parameters"] == ["final_W.prsp", "final_sigma2.prsp", "final_pi.prsp"]
    assert m["tolerance"] is None and m["temperature"] == [[0.0, 1.0]]
    run = rio.Run(str(out))
    assert run.model == "tsc" and run.latents == 8
    ms, mm, ex = run.infer(y[:50])
    g = P.LinearDiscreteGpuModel("tsc", y.shape[1], 8, P.TruncationConfig(8, 5, 3))
    inf = g.inference(P.LinearDiscreteParams(r.params["W"], r.params["sigma2"][0, 0], r.params["pi"][0, 0]), y[:50])
    assert np.array_equal(ms, inf.map_states) and np.array_equal(mm, inf.map_mass)
    assert np.array_equal(ex, inf.expected_states)
    g.close()
    run.close()


@pytest.mark.parametrize("model,values", [("dsc", [-1.0, 0.0, 2.0]), ("mca", None)])
def test_run_directory_other_models(rio, port, tmp_path, model, values):
    y = bars(port, seed=13)
    out = tmp_path / model
    cfg = rio.TrainConfig(model=model, latents=8, hprime=5, gamma=3, values=values, iterations=2, seed=4,
                          tolerance=1e-9, w_noise=[(0.0, 0.1), (1.0, 0.0)])
    r = rio.train(cfg, y, out_dir=str(out))
    m = json.load(open(out / "manifest.json"))
    names = ["W", "sigma2", "values", "probs"] if model == "dsc" else ["W", "sigma2", "pi"]
    assert m["parameters"] == [f"final_{n}.prsp" for n in names]
    assert m["tolerance"] == 1e-9 and m["w_noise"] == [[0.0, 0.1], [1.0, 0.0]]
    if model == "dsc":
        assert m["values"] == values
    run = rio.Run(str(out))
    for n in names:
        assert np.array_equal(run.param(n), r.params[n])
    ms, mm, ex = run.infer(y[:20])
    assert ms.shape == (20, 8) and np.all(mm > 0) and np.all(mm <= 1)
    run.close()
