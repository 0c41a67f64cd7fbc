"""Multi-GPU DAG placement (f2; csrc/multi.cpp) on a B200: two slots backed by
device 0 (the one-GPU box), so every cross-slot edge is a real copy between
two replicas plus cross-slot events, and every result is checked against the
fp64 oracle (B&S 1e-10 relative + 1e-12 absolute; VEC fp32 criteria)."""
import numpy as np
import pytest
import torch

import synth
from oracle import bs as obs
from oracle import vec as ovec
from paper_2012_09646_b200 import dagrt as D

pytestmark = pytest.mark.gpu

BS = (0.08, 0.30, 1.0, 60.0)


def bs_close(out, ref):
    return np.all(np.abs(out - ref) <= 1e-10 * np.abs(ref) + 1e-12)


@pytest.mark.parametrize("placement", ["data", "round_robin"])
def test_bs_from_host_mirrors_over_two_slots(placement):
    """10 B&S vectors from pinned host mirrors: placed over both slots,
    uploaded on the slot that prices them, read back through the slot
    holding each result; a second input set written into the mirrors is
    picked up (uploads of the first set finished before the mirror changed)."""
    n, nv = 300_001, synth.BS_NVEC
    sp = synth.spec_bs(n, nv)
    with D.Multi(devices=[0, 0], placement=placement) as m:
        host = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(nv)]
        S = [m.register_tensor(f"s{i}", mirror=host[i]) for i in range(nv)]
        Cs = [m.register(f"c{i}", 8 * n) for i in range(nv)]
        for set_index in (0, 1):
            seed = synth.BASE_SEED + set_index
            for i in range(nv):
                host[i].numpy()[:] = synth.draw(seed, f"s{i}", sp[f"s{i}"])
                m.write(S[i], host[i].data_ptr())
            placed = [m.launch("bs", 296, 256, S[i], Cs[i], n, *BS) for i in range(nv)]
            assert sorted(set(placed)) == [0, 1]
            for i in range(nv):
                out = np.empty(n, np.float64)
                m.read(Cs[i], out.ctypes.data)
                assert bs_close(out, obs.call(host[i].numpy().astype(np.float64))), (set_index, i)
        st = m.stats()
        assert st["migrations_host"] == 2 * nv and st["per_slot"][0] + st["per_slot"][1] == 2 * nv


def test_vec_chain_across_slots():
    """x1 = x^2 on slot 1 from x resident on slot 0 (peer copy in), y1 = y^2 on
    slot 0, z = sum(x1 - y1) on slot 0 (x1 copied back): the oracle's z."""
    n = 1_000_003
    sp = synth.spec_vec(n)
    seed = synth.BASE_SEED
    xs = synth.draw(seed, "x", sp["x"])
    ys = synth.draw(seed, "y", sp["y"])
    x = torch.from_numpy(xs).cuda()
    y = torch.from_numpy(ys).cuda()
    with D.Multi(devices=[0, 0]) as m:
        X = m.register_tensor("x", x, home=0)
        Y = m.register_tensor("y", y, home=0)
        X1, Y1, Z = m.register("x1", 4 * n), m.register("y1", 4 * n), m.register("z", 8 + 8 * 1024)
        assert m.launch("square", 512, 256, X, X1, n, slot=1) == 1
        assert m.launch("square", 512, 256, Y, Y1, n, slot=0) == 0
        assert m.launch("reduce_diff", 512, 256, X1, Y1, Z, n, slot=0) == 0
        z = np.empty(2, np.float32)
        m.read(Z, z.ctypes.data, 0, 4)
        x1 = np.empty(n, np.float32)
        m.read(X1, x1.ctypes.data)
        ox1, _, oz = ovec.vec(xs, ys)
        rms = np.sqrt(np.mean(ox1 * ox1))
        assert np.all(np.abs(x1 - ox1) <= 1e-4 * np.abs(ox1) + 1e-4 * rms)
        assert abs(z[0] - oz) <= 1e-3 * abs(oz)
        assert m.stats()["migrations_peer"] == 2


def test_overwrite_after_outgoing_copy():
    """WAR across slots on the device: slot 1 squares x (copied from slot 0)
    while slot 0 then overwrites x; slot 1's result is x's OLD square."""
    n = 4_000_000
    x = torch.rand(n, device="cuda")
    w = torch.rand(n, device="cuda")
    old = x.clone()
    with D.Multi(devices=[0, 0]) as m:
        X = m.register_tensor("x", x, home=0)
        W = m.register_tensor("w", w, home=0)
        X1 = m.register("x1", 4 * n)
        m.launch("square", 1184, 256, X, X1, n, slot=1)
        m.launch("square", 1184, 256, W, X, n, slot=0)  # x <- w^2
        got = np.empty(n, np.float32)
        m.read(X1, got.ctypes.data)
        assert np.array_equal(got, (old * old).cpu().numpy())
        m.sync()
        assert torch.equal(x, w * w)
