"""C5 dimension sweep (bench.bench_c5) formatted for profiles/ (never the bench line itself)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

out = bench.bench_c5()
print("# bench.py suite_c5 on B200: CEC2022 F1/F4/F10, ps=10^4, ms per device-loop iteration and rotation TFLOP/s")
print("# dmma: k_cec_eval (D<=104, register-resident m8n8k4 tiles) or the batched GEMM (D=1000); "
      "fma: lane-per-output FMA")
for r in out["rows"]:
    print(f"F{r['fn']:<3} D={r['dim']:<5} {r['rotation']:<6} {r['ms_per_iteration']:8.4f} ms  "
          f"{r['rotation_tflops']:6.2f} TFLOP/s")
