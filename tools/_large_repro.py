import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import test_gpu_parity as T
T.test_large_shapes_use_the_chunked_dp_path()
print("ok")
