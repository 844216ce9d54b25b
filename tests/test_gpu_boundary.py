"""Boundary robustness (include/pscwin.h conventions): concurrent calls on two streams from two host threads give
byte-identical results to sequential calls (the side stream of the pad work and its fork / join events are private
to each thread and device), and a contract error is reported synchronously without touching the outputs."""
import threading

import pytest

import synth
from gpu_util import X_SCALE, dev, dev_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2407_02109_b200 as p
    return p


def test_concurrent_forward_two_streams_two_threads(pl):
    import torch
    cfgs = [synth.vitb(64, cycle_scan=1), synth.vitb(64, B=2)]          # shifted LEARNABLE: the side stream forks
    layers = [pl.PSCWinLayer(pl.LayerDesc.from_config(c), dev_weights(synth.make_weights(c, layer=i), c))
              for i, c in enumerate(cfgs)]
    xs = [dev(synth.make_input(c, layer=i, scale=X_SCALE)) for i, c in enumerate(cfgs)]
    ref = [layer(x).clone() for layer, x in zip(layers, xs)]
    torch.cuda.synchronize()
    n_iter = 20
    outs = [[None] * n_iter for _ in cfgs]
    errors = []

    def worker(j):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for i in range(n_iter):
                    outs[j][i] = layers[j](xs[j])
            s.synchronize()
        except Exception as e:  # surfaced in the main thread
            errors.append(e)

    th = [threading.Thread(target=worker, args=(j,)) for j in range(len(cfgs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for j in range(len(cfgs)):
        for i in range(n_iter):
            assert torch.equal(outs[j][i], ref[j]), (j, i)


def test_contract_error_is_synchronous(pl):
    import torch
    cfg = synth.tiny(H=12, W=12, shift_x=0, shift_y=0)                  # 12 % 8 != 0: plain windows need divisibility
    layer_cfg = synth.tiny()
    w = dev_weights(synth.make_weights(layer_cfg), layer_cfg)
    with pytest.raises(pl.PscwinError):
        pl.PSCWinLayer(pl.LayerDesc.from_config(cfg), w)(torch.zeros(1, 12, 12, 64, dtype=torch.bfloat16,
                                                                        device="cuda"))
