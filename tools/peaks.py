"""FP64 throughput microbenchmarks on the device (DFMA loop, DMMA m8n8k4 loop, both)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_05186_b200 as pb  # noqa: E402

out = {}
for mode, name in [(0, "dfma"), (1, "dmma_m8n8k4"), (2, "dfma+dmma")]:
    out[name + "_tflops"] = max(pb.fp64_peak(0, mode=mode) for _ in range(3)) / 1e12
print(json.dumps(out))
