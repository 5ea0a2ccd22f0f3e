"""Stream-form knobs (emit_stream module constants: ZCHUNK, TJ, PD, NSTG ...) against the
hand-tuned kernel: python scripts/stream_knob_probe.py 768 ZCHUNK=96 [TJ=32 ...]"""
import sys, runpy
sys.path.insert(0, ".")
from paper_1907_02818_b200 import emit_stream
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    setattr(emit_stream, k, int(v) if v.lstrip('-').isdigit() else v)
sys.argv = ["emitted_time.py", sys.argv[1]]
runpy.run_path("scripts/emitted_time.py", run_name="__main__")
