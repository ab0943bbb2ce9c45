"""Quick GPU probe: parity on C1 + lattice stress set, timing on larger inputs."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2411_09809_b200 as G
from paper_2411_09809_b200 import configs, metrics as M
from oracle import glare_oracle as O, sweep as S

res = {}
g, p = configs.config1()
t = time.time()
out = dict(nc=G.node_occlusion(g, p['radius']), ma=G.minimum_angle(g), ml=G.edge_length_variation(g),
           ec=G.edge_crossing(g), scan=G._crossing_scan(g, p['ideal']), eca=G.edge_crossing_angle(g, p['ideal']))
print('C1 gpu', out, time.time() - t, flush=True)
print('C1 want nc=159 ma=0.06463926772041739 ml=0.006660526515776418 ec=2965010 dev=1033395.8742814541 eca=0.7147240545921593')

rng = np.random.default_rng(7)
xy = rng.integers(0, 64, (3000, 2)).astype(np.float64)
pairs = rng.integers(0, 3000, (6000, 2))
pairs = pairs[np.any(xy[pairs[:, 0]] != xy[pairs[:, 1]], axis=1)]
gl = G.LayoutGraph(np.arange(3000), xy, pairs)
out = dict(m=gl.num_edges, nc=G.node_occlusion(gl, 1.0), ma=G.minimum_angle(gl), ml=G.edge_length_variation(gl),
           scan=G._crossing_scan(gl, configs.IDEAL_70))
print('lattice gpu', out, flush=True)
print('lattice want m=5992 nc=9588 ma=0.22813915546418073 ml=0.00614032561565724 ec=4194903 dev=1475177.8703388437')

g2, p2 = configs.config2()
t = time.time(); c_or = S.crossing_scan(g2.xy, g2.edges, p2['ideal']); print('C2 C-oracle', c_or, time.time() - t, flush=True)
t = time.time(); c_gpu = G._crossing_scan(g2, p2['ideal']); torch.cuda.synchronize(); print('C2 gpu', c_gpu, time.time() - t, flush=True)
print('C2 nc', G.node_occlusion(g2, p2['radius']), S.node_occlusion(g2.xy, p2['radius']))
print('C2 ma', G.minimum_angle(g2), O.minimum_angle(g2.xy, g2.edges))
print('C2 ml', G.edge_length_variation(g2), O.edge_length_variation(g2.xy, g2.edges))

# timing: synthetic uniform segments
for m in (200_000, 1_000_000):
    n = 2 * m
    xy = np.random.default_rng(3).uniform(0, 1, (n, 2))
    e = np.stack([np.arange(0, n, 2), np.arange(1, n, 2)], 1)
    gg = G.LayoutGraph.from_normalized(xy, e)
    dg = M.DeviceGraph.from_graph(gg)
    rec = M.CrossingRecords(dg)
    print('fast path', rec.fast_path())
    for ideal in (None, configs.IDEAL_70):
        rec.partial(ideal, 0, rec.units); torch.cuda.synchronize()
        s, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); out = rec.partial(ideal, 0, rec.units); e_.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e_); pairs = m * (m - 1) / 2
        print(f'm={m} angle={ideal is not None} {ms:.2f} ms {pairs/ms/1e9:.3f} Tpairs/s count={out[0].item():.0f}', flush=True)
    thr = M.occlusion_threshold(1e-4)
    M.occlusion_partial(dg, thr, 0, M.occlusion_units(n)); torch.cuda.synchronize()
    s.record(); o = M.occlusion_partial(dg, thr, 0, M.occlusion_units(n)); e_.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e_); pairs = n * (n - 1) / 2
    print(f'occ n={n} {ms:.2f} ms {pairs/ms/1e9:.3f} Tpairs/s count={o.item():.0f}', flush=True)
