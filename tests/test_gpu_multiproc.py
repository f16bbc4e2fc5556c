"""Two ranks, one GPU: tile-band rendering with the peer-memory output (CUDA IPC) must reproduce the
single-process frame bit for bit.  (gpurun exposes one B200; two processes on it exercise the same IPC
mapping that two GPUs of one box use over NVLink, with gloo for the control messages.)"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2505_24796_b200 as tcgs
    from paper_2505_24796_b200 import shard, synthetic

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        scene = synthetic.gen_uniform(60000, 640, 360, seed=21)
        cam = synthetic.make_camera(640, 360)
        cloud = tcgs.GaussianCloud.from_arrays(scene, "cuda")
        br = shard.BandRenderer("cuda", output="peer")
        cam2 = synthetic.CameraSpec(cam.view, cam.fx * 1.1, cam.fy * 1.1, cam.cx, cam.cy, cam.width, cam.height,
                                    cam.near)
        cams = [cam, cam2, cam]
        results = []
        prev = None
        for k, c in enumerate(cams):  # three frames, two cameras: the mapping and both slots are reused
            bf = br.render(cloud, c, with_stats=True)
            if rank == 0:
                ref = tcgs.Renderer("cuda").render_frame(cloud, c, timed=False)
                results.append((torch.equal(bf.rgb, ref.rgb), torch.equal(bf.T, ref.T),
                                torch.equal(bf.n_contrib, ref.n_contrib),
                                bf.stats.f_blend == ref.stats.f_blend, bf.stats.n_splats == ref.stats.n_splats,
                                bf.bands))
                if prev is not None:  # double buffering: the previous frame is still intact on rank 0
                    results.append(tuple([torch.equal(prev[0], prev[1])] * 5) + (bf.bands,))
                prev = (bf.rgb, ref.rgb.clone())
        br.close()
        if rank == 0:
            q.put(results)
    finally:
        dist.destroy_process_group()


def test_peer_band_output_two_ranks_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for rgb_eq, t_eq, n_eq, blend_eq, n_eq2, bands in res:
        assert len(bands) == 2 and bands[0][0] == 0 and bands[1][1] == (360 + 15) // 16
        assert rgb_eq and t_eq and n_eq and blend_eq and n_eq2
