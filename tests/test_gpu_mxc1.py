"""GPU: the MXC1 container on the device (SURVEY.md §8(f)4,
mx/codec.py:287-380).  serialize_device writes exactly the bytes of the
host serialize (which equal the reference's, tests/test_codec_golden);
deserialize_device raises the same exceptions as deserialize on the same
malformed containers and round-trips to identical streams and decodes."""

import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.golden import inputs  # noqa: E402


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch.device("cuda", 0)


SHAPES = [(), (1,), (7,), (33,), (4, 1000), (3, 5, 7), (2, 3, 4, 5), (0,), (2, 0, 3),
          (1, 64, 512)]
SPECS = ["fp4_e2m1:32:e8m0", "fp5_e2m2:16:e5m0", "fp3_e1m1:8:e5m0", "int4:64:e8m0",
         "fp4_e2m1:24:e4m0", "int8:32:e8m0"]


def test_serialize_device_matches_host(cuda):
    from paper_2411_09510_b200 import (compress_tensor, compress_tensor_device, parse_scheme,
                                       serialize, serialize_device)
    from paper_2411_09510_b200.formats import ELEMENT_CODES

    for spec in SPECS:
        sch = parse_scheme(spec, extensions=True)
        if sch.element.name not in ELEMENT_CODES:
            continue
        for shape in SHAPES:
            n = int(np.prod(shape)) if shape else 1
            x = inputs.gauss_f32(n, 11 + n).astype(np.float32).reshape(shape)
            host = serialize(compress_tensor(x, sch))
            dct = compress_tensor_device(torch.from_numpy(x).to(cuda), sch)
            dev = serialize_device(dct)
            assert dev.is_cuda and dev.dtype == torch.uint8
            assert dev.cpu().numpy().tobytes() == host, (spec, shape)


def test_roundtrip_device(cuda):
    from paper_2411_09510_b200 import (compress_tensor_device, decompress_tensor_device,
                                       deserialize, deserialize_device, parse_scheme,
                                       serialize_device)

    sch = parse_scheme("fp4_e2m1:32:e8m0")
    for shape in [(2048, 4096), (3, 5, 7), (1,)]:
        n = int(np.prod(shape))
        x = torch.from_numpy(inputs.gauss_bf16(n, 5).astype(np.float32).reshape(shape)).to(
            cuda, torch.bfloat16)
        dct = compress_tensor_device(x, sch)
        buf = serialize_device(dct)
        for copy in (True, False):
            back = deserialize_device(buf, copy=copy)
            assert back.scheme == sch and tuple(back.shape) == tuple(shape)
            assert torch.equal(back.scale, dct.scale) and torch.equal(back.elements, dct.elements)
            a = decompress_tensor_device(back, torch.float32)
            b = decompress_tensor_device(dct, torch.float32)
            assert torch.equal(a, b)
        host = deserialize(buf.cpu().numpy().tobytes())
        assert host.scale_stream == dct.scale.cpu().numpy().tobytes()


def test_deserialize_device_errors_match_host(cuda):
    from paper_2411_09510_b200 import (compress_tensor, deserialize, deserialize_device,
                                       parse_scheme, serialize)

    good = serialize(compress_tensor(np.arange(100, dtype=np.float32), parse_scheme(
        "fp4_e2m1:32:e8m0")))
    bad = [
        b"", good[:10], b"XXC1" + good[4:],                   # truncated / magic
        good[:4] + bytes([2]) + good[5:],                     # version
        good[:7] + bytes([1]) + good[8:],                     # flags
        good[:4] + good[4:6] + bytes([99]) + good[7:],        # scale code
        good[:4] + good[4:5] + bytes([0xF0]) + good[6:],      # format code (TopK)
        good[:8] + struct.pack("<I", 0) + good[12:],          # block size 0
        good[:-1], good + b"\0",                              # payload length
        good[:16] + struct.pack("<I", 3) + good[20:],         # reserved field
        good[:12] + struct.pack("<I", 300) + good[16:],       # ndim beyond the data
    ]
    for data in bad:
        with pytest.raises(Exception) as host_exc:
            deserialize(data)
        t = torch.from_numpy(np.frombuffer(data, dtype=np.uint8).copy()).to(cuda)
        with pytest.raises(Exception) as dev_exc:
            deserialize_device(t)
        assert type(dev_exc.value) is type(host_exc.value), (data[:24], host_exc.value,
                                                              dev_exc.value)


def test_serialize_device_graph_capturable(cuda):
    from paper_2411_09510_b200 import (compress_tensor_device, parse_scheme, serialize,
                                       serialize_device)

    sch = parse_scheme("fp4_e2m1:32:e8m0")
    x = torch.randn(4096, 1024, device=cuda).to(torch.bfloat16)
    dct = compress_tensor_device(x, sch)
    out = serialize_device(dct).clone()
    out.zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        serialize_device(dct, out=out)
    g.replay()
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == serialize(dct)
