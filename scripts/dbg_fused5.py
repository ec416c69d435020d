import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from paper_2505_20839_b200 import fireq
fireq.load()
import test_gpu_ffn as T
try:
    T.test_fused_ffn_llama2_7b(fireq)
    print("PASS")
except AssertionError as e:
    import traceback; traceback.print_exc()
