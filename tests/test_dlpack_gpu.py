"""Zero-copy device views: the reference copies every
result into a NumPy array (proj/python/bindings.cpp:25-42); here amplitudes,
probabilities and rho are exported in place through DLPack and
__cuda_array_interface__, and the exported memory is the state's own."""
import gc

import numpy as np
import pytest

from paper_2401_06861_b200 import abi

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_sv_amplitudes_dlpack_zero_copy(port):
    n = 12
    ops = port.random_circuit(31, n, 80)
    sv = abi.SV(n)
    sv.apply(ops)
    view = sv.device_view()
    assert view.__dlpack_device__() == (2, 0)
    t = torch.from_dlpack(view)
    assert t.dtype == torch.complex128 and t.shape == (1 << n,) and t.is_cuda
    assert t.data_ptr() == view.ptr  # same HBM, no copy
    np.testing.assert_array_equal(t.cpu().numpy(), sv.amplitudes())
    np.testing.assert_allclose(t.cpu().numpy(), port.sv_run(n, ops), atol=1e-10, rtol=0)
    # __cuda_array_interface__ consumers see the same memory
    t2 = torch.as_tensor(view, device="cuda")
    assert t2.data_ptr() == view.ptr


def test_sv_probabilities_on_device_match_host_bits(port):
    n = 14
    ops = port.random_circuit(32, n, 100)
    sv = abi.SV(n)
    sv.apply(ops)
    p = torch.from_dlpack(sv.device_probabilities())
    assert p.dtype == torch.float64 and p.shape == (1 << n,)
    host = sv.probabilities()
    np.testing.assert_array_equal(p.cpu().numpy(), host)
    a = sv.amplitudes()
    # |a|^2 rounded as std::norm (re*re + im*im, no FMA): bit-identical
    np.testing.assert_array_equal(host, a.real * a.real + a.imag * a.imag)


def test_view_keeps_owner_alive():
    t = torch.from_dlpack(abi.SV(10).device_view())  # the temporary state lives as long as the tensor
    gc.collect()
    assert t[0].item() == 1.0 and float(t.abs().sum()) == 1.0


def test_dm_rho_and_probabilities_dlpack(port):
    n = 5
    ops = port.random_circuit(33, n, 40)
    dm = abi.DM(n)
    dm.apply(ops)
    dm.apply_channel([1], port.depolarizing(0.1))
    rho = torch.from_dlpack(dm.device_view())
    assert rho.shape == (1 << n, 1 << n)
    np.testing.assert_array_equal(rho.cpu().numpy(), dm.rho())
    p = torch.from_dlpack(dm.device_probabilities())
    np.testing.assert_array_equal(p.cpu().numpy(), dm.probabilities())


def test_large_dm_view_is_row_major_after_mirror_passes(port):
    # n = 9 density matrices run in the interleaved layout with Hermitian
    # mirror passes; the exported view is the reference's row-major rho
    n = 9
    ops = port.random_circuit(34, n, 60, 2)
    dm = abi.DM(n)
    dm.apply(ops)
    got = torch.from_dlpack(dm.device_view()).cpu().numpy()
    want = port.dm_run(n, ops)
    np.testing.assert_allclose(got, want, atol=1e-10, rtol=0)
