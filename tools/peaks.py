"""Prints the device microbenchmark peaks used as roofline denominators."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09501_b200 as p3s
p3s.set_device(0)
print("smem contiguous GB/s %.0f" % (p3s.smem_peak(False) / 1e9))
print("smem gather GB/s %.0f" % (p3s.smem_peak(True) / 1e9))
print("fp64 non-FMA Gop/s %.0f" % (p3s.fp64_peak() / 1e9))
