#!/usr/bin/env python3
"""Probe: cudaMemcpy2DAsync between pinned host memory and the device as a
function of the row width (the host path's slab copies are 2D copies whose
rows get narrower as a transposition is cut into more slabs).

    python scripts/copy2d_probe.py
"""
import ctypes as C
import torch


def main():
    rt = C.CDLL("libcudart.so")
    rt.cudaMemcpy2DAsync.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_size_t,
                                     C.c_size_t, C.c_int, C.c_void_p]
    total = 1 << 30
    h = torch.empty(2 * total, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(2 * total, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    s = torch.cuda.current_stream().cuda_stream
    for kind, name in ((1, "H2D"), (2, "D2H")):
        for width, pitch in ((1 << 11, 0), (1 << 12, 0), (1 << 14, 0), (1 << 16, 0), (1 << 20, 0), (1 << 24, 0),
                             (5224, 167184), (5224, 5224 * 32), (20896, 167184), (41792, 167184),
                             (4104, 8208), (65528, 131064)):
            pitch = pitch or 2 * width
            height = min(total // width, (2 * total) // pitch)
            dst, src = (d, h) if kind == 1 else (h, d)
            best = 1e30
            for _ in range(3):
                e0.record()
                done = 0
                while done < height:  # the runtime limits the height of one call
                    hh = min(32768, height - done)
                    off = done * pitch
                    rc = rt.cudaMemcpy2DAsync(dst.data_ptr() + off, pitch, src.data_ptr() + off, pitch,
                                              width, hh, kind, s)
                    assert rc == 0, rc
                    done += hh
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(f"{name} rows of {width:>9d} bytes at pitch {pitch:>9d}: "
                  f"{width * height / 1e9 / (best / 1e3):6.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
