import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_10859_b200 as wv
from paper_2208_10859_b200 import _native as N
path = os.path.join('tests', 'golden', sys.argv[1] if len(sys.argv) > 1 else 'golden_quantized.wvv')
s = wv.DecodeSession(path)
lib = N.load()
mode = sys.argv[2] if len(sys.argv) > 2 else "full"
h = s.header
mask = wv.stereo_mask(wv.CameraPose(yaw=30, pitch=10), (h.mask_w, h.mask_h)) if h.stereo else wv.viewport_to_mask(wv.CameraPose(yaw=30, pitch=10), (h.mask_w, h.mask_h))
args = s._mode_args(mode, mask, wv.FoveationSchedule.default(h.levels), 0)
dev, ext, _ = s._make_resident(0)
e, _, _ = s._entry_for(0)
args.t = 0; args.d_payload = dev.data_ptr(); args.payload_bytes = dev.numel(); args.d_extrema = ext.data_ptr()
args.d_set_loaded = e.loaded.data_ptr(); args.d_set_bytes = e.nbytes.data_ptr(); args.d_canvas = s._canvas.data_ptr()
args.d_footprint = s._footprint.data_ptr(); args.d_result = s._results[0].data_ptr()
g, ws, cs = C.byref(s._geom), C.c_void_p(s._ws.data_ptr()), C.c_void_p(s.stream.cuda_stream)
for name in ("wv_select", "wv_dequant_temporal", "wv_synthesize"):
    st = getattr(lib, name)(g, C.byref(args), ws, cs)
    print(name, "status", st, flush=True)
    try:
        s.stream.synchronize(); print(name, "ok", flush=True)
    except Exception as ex:
        print(name, "FAILED", str(ex)[:200], flush=True); break
