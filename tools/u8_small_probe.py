"""Single-frame probe: graph replay of a ring of frames (u8 or f32) under the current HARRIS_DEV
knobs (HARRIS_U8_CONFIG / HARRIS_TMA_CONFIG / HARRIS_BAND_ROWS); us per frame.
python tools/u8_small_probe.py H W [f32]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

H, W = int(sys.argv[1]), int(sys.argv[2])
u8 = not (len(sys.argv) > 3 and sys.argv[3] == "f32")
modes = tuple(sys.argv[4].split(",")) if len(sys.argv) > 4 else ("graph",)
r = bench.frame_stream(H, W, 180, u8=u8, modes=modes)
for mode in modes:
    print(json.dumps({"u8": u8, "HW": [H, W], "mode": mode, "share": os.environ.get("HARRIS_STREAM_SHARE"),
                      "us": round(r[mode]["us_per_frame"], 2), "frac": round(r[mode]["frac_of_measured_hbm"], 3),
                      "identical": r[mode]["outputs_identical"]}))
raise SystemExit(0)
print(json.dumps({"u8": u8, "HW": [H, W], "cfg": os.environ.get("HARRIS_U8_CONFIG" if u8 else "HARRIS_TMA_CONFIG"),
                  "band": os.environ.get("HARRIS_BAND_ROWS"),
                  "us": r["graph"]["us_per_frame"], "frac": r["graph"]["frac_of_measured_hbm"]}))
