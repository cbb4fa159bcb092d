"""Print the float32 bit patterns of q / 255 (numpy float32 division, the
reference's dequantize_values) for csrc/wv_temporal.cu's kQ255Bits."""
import numpy as np

v = (np.arange(256, dtype=np.float32) / np.float32(255.0)).view(np.uint32)
for i in range(0, 256, 8):
    print("    " + ", ".join(f"0x{x:08x}u" for x in v[i:i + 8]) + ",")
