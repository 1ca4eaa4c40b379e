"""NEXT-3 (safety-rule validation) and NEXT-2 (colouring) on the GPU path."""
import pytest

import me_inputs as mi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def me():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2411_06465_b200 import build
    build.build()
    import paper_2411_06465_b200 as me
    return me


def measured_runs():
    """The paper's 454 measured outcomes."""
    out = []
    for r in mi.load_paper_tables():
        if r["kind"] != "thr":
            continue
        N, t, c, p = r["n_gpus"], r["tp"], r["cp"], r["pp"]
        out.append(dict(model_shape=mi.PRESETS[r["model"]], d=N // (t * c * p), t=t, p=p, c=c, b=r["mbs"],
                        s=r["seq"], gbs=1024, cap_gb=r["gpu_gb"], oom=r["text"] == "OOM", paper_colour=r["colour"],
                        line=r["line"]))
    return out


def test_safety_rule_confusion(me, oracle_mod):
    from paper_2411_06465_b200 import validate
    runs = measured_runs()
    cl = validate.classify(runs)
    assert all(r["colour"] == r["paper_colour"] for r in cl)
    for r in cl[::37]:
        e = oracle_mod.estimate(r["model_shape"], d=r["d"], t=r["t"], p=r["p"], c=r["c"], b=r["b"], s=r["s"],
                                gbs=1024)
        assert e["total"] == r["total"]
    assert validate.confusion(cl) == {("green", False): 207, ("yellow", False): 34, ("yellow", True): 42,
                                      ("red", True): 171}
    rep = validate.report(runs)
    assert rep["rule_holds"] and rep["green_oom"] == 0 and rep["red_trained"] == 0
