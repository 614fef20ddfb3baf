"""Phase timeline of single tcgen05-engine launches (diagnostics). For each launch index n of one
actor forward+backward at the given config, re-run in a fresh process with SPIKERL_TC_TRACE=n and
print the %globaltimer stamps of CTA 0 relative to its entry (ns):
  1 setup done  2 first TMA issued  3 first full stage  4 first accumulator committed
  6 epilogue got accumulator  7 epilogue done (unit 0)  8 teardown start  9 TMEM freed
  10 FWD epilogue: first TMEM load back  11 FWD epilogue: scan done"""
import os, sys, subprocess, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def child(name, B, n):
    import numpy as np, torch
    import synthgen as sg
    import paper_2502_17496_b200 as pk
    from paper_2502_17496_b200 import _lib
    shape, _, _ = sg.preset(name)
    rng = np.random.default_rng(0)
    p = sg.actor_params(shape, rng)
    a = pk.SpikingActor(pk.actor_cfg_from(shape), B)
    a.load(p)
    s = torch.from_numpy(sg.observations(rng, B, shape.obs_dim)).cuda()
    g = torch.from_numpy(sg.action_grads(rng, B, shape.act_dim)).cuda()
    for _ in range(2):   # the second (warm) iteration's launches are the traced ones
        a.forward(s); a.backward(s, g)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)()
    _lib.lib().spikerl_debug_tc_trace(buf)
    v = list(buf)
    print(json.dumps({"n": n, "stamps": [(x - v[0]) if x else None for x in v]}))

if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4])); sys.exit(0)
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    for n in range(1, 10):
        env = dict(os.environ, SPIKERL_TC_TRACE=str(n + 9))
        r = subprocess.run([sys.executable, __file__, "--child", name, str(B), str(n)], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-400:])
