import subprocess, sys, os
CODE = open(os.path.join(os.path.dirname(__file__), "debug_tma.py")).read().split("CODE = r'''")[1].split("'''")[0]
for dbg in ["0", "1", "2", "3"]:
    for case in [("float32", "fp32", "64", "64", "4", "4"), ("float64", "fp64", "130", "130", "6", "6")]:
        env = dict(os.environ, SWDFT2D_DBG=dbg, CUDA_LAUNCH_BLOCKING="1")
        r = subprocess.run([sys.executable, "-c", CODE, *case], capture_output=True, text=True, env=env, timeout=120)
        msg = r.stdout.strip().splitlines()[-1:] if r.returncode == 0 else [l for l in r.stderr.splitlines() if "CUDA error" in l or "Error" in l][:1]
        print("dbg", dbg, case, r.returncode, msg, flush=True)
