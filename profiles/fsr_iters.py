"""fsr_batch4 iterations / events per pixel on sampled pixels of a scene (host build of the automaton): python profiles/fsr_iters.py SCENE W H T"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2412_11639_b200 as spk
h = C.CDLL("/root/repo/tests/native/libfsm_host.so")
h.batch_iters.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p]
scene, W, H, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
v = spk.synth(scene, 0, W, H, T, device="cuda")
pl = v.planes.cpu().numpy()
rng = np.random.default_rng(0)
its, evs, spk_ = [], [], []
for p in rng.choice(W * H, 200, replace=False):
    bits = ((pl[:, p >> 3] >> (p & 7)) & 1).astype(np.uint8)
    it, ev = C.c_long(), C.c_long()
    h.batch_iters(bits.ctypes.data, T, C.byref(it), C.byref(ev))
    its.append(it.value); evs.append(ev.value); spk_.append(int(bits.sum()))
print(scene, "words", (T + 31) // 32, "iters mean", np.mean(its), "max", max(its),
      "events mean", np.mean(evs), "spikes mean", np.mean(spk_))
