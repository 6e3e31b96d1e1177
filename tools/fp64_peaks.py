"""FP64 roofline denominators: cuBLAS DGEMM burst/sustained + DMMA/DFMA loops."""
import json, subprocess, time, os, sys
import torch

def dgemm(n=8192, seconds=4.0):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n**3 / (best * 1e-3) / 1e12
    t0 = time.time(); k = 0
    e0.record()
    while time.time() - t0 < seconds:
        c = a @ b; k += 1
        if k % 4 == 0: torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sust = 2 * n**3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return burst, sust

if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    out = {}
    clk_log = open("gpurun_out/fp64_clocks.csv", "w")
    clk = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader", "-lms", "200"], stdout=clk_log, text=True)
    b, s = dgemm()
    out["cublas_dgemm_8192_burst_tflops"] = b
    out["cublas_dgemm_8192_sustained_tflops"] = s
    r = subprocess.run([os.path.join(os.path.dirname(__file__), "fp64_peaks")], capture_output=True, text=True)
    out["micro"] = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    clk.kill()
    clk.wait()
    clk_log.close()
    out["clock_samples"] = open("gpurun_out/fp64_clocks.csv").read().splitlines()[-40:]
    print(json.dumps(out, indent=1))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/fp64_peaks.json", "w"), indent=1)
