"""Small-path cases one by one (each in its own process under a short timeout)."""
import os, subprocess, sys
CASES = {
    "n2": "X = np.random.default_rng(0).normal(size=(2, 3))",
    "n3": "X = np.random.default_rng(0).normal(size=(3, 3))",
    "n129": "X = np.random.default_rng(0).normal(size=(129, 3))",
    "n2049": "X = np.random.default_rng(0).normal(size=(2049, 3))",
    "ties3000": "X = np.random.default_rng(0).integers(-3, 4, size=(3000, 6)).astype(np.float64)",
    "c1": "from paper_1402_3789_b200.datagen import config_dataset; X = config_dataset('c1')",
    "dmax": "X = np.random.default_rng(0).normal(size=(3000, 5)); kw = dict(dmax=0.5)",
    "kl1": "X = np.random.default_rng(0).normal(size=(3000, 5)); kw = dict(kl1=40)",
}
mode = sys.argv[1] if len(sys.argv) > 1 else "2"
for name, setup in CASES.items():
    code = ("import numpy as np, time, paper_1402_3789_b200 as nnm\nkw = {}\n" + setup +
            "\nfrom oracle import nnm_oracle as orc\nt=time.time(); r = nnm.fit(X, **kw); t=time.time()-t\n"
            "m, a = orc.single_linkage(X, **kw)\n"
            "ok = all(np.array_equal(r.merges.array[f], m[f]) for f in ('root_a','root_b','dist','new_size','point_a','point_b')) and np.array_equal(r.assignments, a)\n"
            "print(len(X), r.rounds, round(t*1e3,1), r.device_stats['scan_ms'], 'OK' if ok else 'MISMATCH')")
    env = dict(os.environ, NNM_SMALL=mode)
    try:
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=60)
        print(name, p.stdout.strip(), p.stderr.strip()[-300:], flush=True)
    except subprocess.TimeoutExpired:
        print(name, "TIMEOUT", flush=True)
