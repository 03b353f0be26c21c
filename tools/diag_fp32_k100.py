import sys; sys.path.insert(0, '.')
import numpy as np, oracle as orc, paper_2503_18118_b200 as xl
orc.build()
K, D = 100, 6
nl = [1024, 2048, 6000, 12000]
a, ao = xl.Array.ula(max(nl), 100e9), orc.array("ula", n_y=max(nl), fc_hz=100e9)
pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=9)
rec = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
res = xl.saturation_sweep(a, nl, K, D, [0.0, 10.0], rec, pos=pos, precision=xl.FP32, per_drop=True)
erg, nv, _, pd = orc.saturation_sweep(ao, nl, pos.cpu().numpy(), [0.0, 10.0], rec, per_drop=True)
g = res["per_drop"].cpu().numpy()
e = g - pd   # D, nN, S, R
np.set_printoptions(precision=2, linewidth=200)
print("max |err| per level x snr x receiver (CAP ZF MMSE MRC):")
print(np.nanmax(np.abs(e), axis=0))
print("mean err:")
print(np.nanmean(e, axis=0))
# gram-level
for N in nl:
    a1, ao1 = xl.Array.ula(N, 100e9), orc.array("ula", n_y=N, fc_hz=100e9)
    G = xl.gram_exact(a1, pos, precision=xl.FP32).cpu().numpy()
    Go = orc.gram_exact(ao1, pos.cpu().numpy())
    d = np.real(np.diagonal(Go, axis1=1, axis2=2))
    bias = np.mean(np.real(np.diagonal(G, axis1=1, axis2=2)) / d - 1)
    sc = np.sqrt(np.abs(d[:, :, None] * d[:, None, :]))
    print(N, "norm err", np.max(np.abs(G - Go) / sc), "diag bias", bias)
