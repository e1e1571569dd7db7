"""F4: a GPU trace drives the reference CLI, and the CLI's placement drives the GPU.

Three origins' batches run through a live B200 layer; their routing is exported
with `B200MoELayer.trace_records` as the reference's activation trace (JSON
lines, reference cli.py:91-135).  `moeplace place` (cmd_place, cli.py:290-318)
runs in-process on a config whose initial statistics come from that trace
(cli.py:275-285).  Checks: exit code 0; the statistics the CLI parsed equal the
GPU's fused histogram; the placement it wrote equals `build_placement("ours")`
on the GPU counts; and, read back as a GPU route table, it gives remote
invocations equal to the reference's `remote_volume` (cost.py:120-129).
"""

import json

import numpy as np
import pytest

from oracle import moe_oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_gpu_trace_through_moeplace_place(tmp_path):
    from paper_2508_12851_b200.errors import import_moeplace
    from paper_2508_12851_b200.layer import B200MoELayer
    from paper_2508_12851_b200.routing import gpu_expert_sets, route_table_for
    from paper_2508_12851_b200.shapes import LayerShape
    from paper_2508_12851_b200.trace import write_trace
    mp = import_moeplace()
    if mp is None:
        pytest.skip("the reference package is not importable here")
    from moeplace.cli import EXIT_OK, load_config, main

    shape = LayerShape("toy_trace", d=512, f=512, E=8, k=2)
    S, T, seed = 3, 256, 13
    experts = {e: orc.synthetic_expert(e, shape.d, shape.f, seed) for e in range(shape.E)}
    wg = orc.synthetic_router(shape.E, shape.d, seed)
    src = lambda e: tuple(torch.from_numpy(w) for w in experts[e])
    layer = B200MoELayer(shape, max_tokens=T, cap_slots=shape.E)
    layer.set_placement_sets([list(range(shape.E))], src)
    trace = tmp_path / "gpu_trace.jsonl"
    counts = np.zeros((S, shape.E), np.int64)
    for s in range(S):                     # origin s's batch, its own routing skew
        layer.set_router(torch.from_numpy(wg), torch.from_numpy(orc.origin_bias(s, shape.E, seed)))
        layer.reset_counts()
        layer.forward(torch.from_numpy(orc.synthetic_tokens(s, T, shape.d, seed)).cuda().bfloat16())
        torch.cuda.synchronize()
        counts[s] = layer.activation_counts()
        write_trace(str(trace), layer.trace_records(T, layer=0, t=float(s), server=s), append=s > 0)

    m_e = shape.expert_bytes
    cluster = {"servers": [{"gpus": [{"memory": 4 * m_e, "load_bandwidth": 770e9}]} for _ in range(S)],
               "link_bandwidth": np.full((S, S), 770e9).tolist(),
               "link_latency": (np.full((S, S), 3e-6) - np.diag(np.full(S, 3e-6))).tolist()}
    model = {"num_layers": 1, "experts_per_layer": shape.E, "top_k": shape.k, "expert_size": m_e,
             "hidden_width": shape.d, "bytes_per_element": 2}
    config = {"cluster_path": "cluster.json", "model_path": "model.json", "strategy": "ours", "seed": 0,
              "output_dir": str(tmp_path / "out"),
              "workload": {"servers": {"mean_interarrival": 1.0, "requests": 4, "tokens": 1,
                                       "selection": "dirichlet", "dirichlet_alpha": 0.3}},
              "initial_stats": {"source": "trace", "path": "gpu_trace.jsonl"}}
    for name, doc in (("cluster.json", cluster), ("model.json", model), ("config.json", config)):
        (tmp_path / name).write_text(json.dumps(doc))
    cfg_path = str(tmp_path / "config.json")
    assert main(["place", "--config", cfg_path]) == EXIT_OK

    cfg = load_config(cfg_path)
    assert np.array_equal(cfg.initial_stats.counts[:, 0, :shape.E], counts)   # CLI parsed the GPU histogram
    doc = json.loads((tmp_path / "out" / "placement.json").read_text())
    stats = mp.ActivationStats.from_counts(counts.astype(float)[:, None, :], (shape.E,))
    ref = mp.build_placement("ours", cfg.cluster, cfg.model, stats, 0)
    assert gpu_expert_sets(doc, 0) == gpu_expert_sets(ref, 0)
    placement = mp.Placement.from_dict(doc, cfg.cluster, cfg.model)
    assert mp.validate_placement(placement, cfg.cluster, cfg.model).ok
    layer.close()

    # the CLI's placement document as the GPU route table: the remote invocations our accounting
    # derives from the GPU counts equal the reference's remote_volume of that placement
    from paper_2508_12851_b200.routing import dispatch_accounting
    route = route_table_for(doc, cfg.cluster, shape.E, shape.d)
    acc = dispatch_accounting(counts, route, shape.d)
    assert acc["remote_invocations"] == mp.remote_volume(placement, stats)
