"""Single-frame stream (the thesis measured one frame at a time):
back-to-back UNBATCHED launches over a ring of K distinct frames (ring > L2, so every frame
streams from HBM), in four launch modes:
  plain        stream-ordered launches
  pdl          programmatic dependent launch (prologue overlaps the previous frame's tail,
               griddepcontrol.wait before touching memory)
  independent  PDL, frames declared independent (no wait: a frame's CTAs take the SMs the
               previous frame has left)
  graph        the ring's K launches (independent mode) captured once in a CUDA graph and
               replayed (no host launch cost)
  frames       harris_run_frames: the whole ring in ONE C call (frame 0 PDL-waits, frames
               1.. independent), still one kernel launch per frame
  frames_graph harris_run_frames captured in a CUDA graph and replayed
Per mode: us per frame (CUDA events over N frames / N), MP/s, fraction of measured HBM.
    python tools/frame_stream.py [frames_per_mode]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2212_12035_b200 as hb  # noqa: E402


if __name__ == "__main__":
    import bench
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 240
    out = {}
    for H, W in [(1536, 2560), (2560, 1536), (2832, 4256), (4256, 2832)]:
        out[f"{W}x{H}"] = bench.frame_stream(H, W, n)
    print(json.dumps(out, indent=1))
