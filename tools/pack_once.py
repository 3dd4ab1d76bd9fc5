import sys; sys.path.insert(0, '.')
import torch
from paper_2505_11076_b200 import _lib
rows, cols = 11008, 4096
g = torch.Generator(device="cuda"); g.manual_seed(0)
for dt in (torch.float16, torch.float32):
    dense = (torch.randint(0, 2, (rows, cols), generator=g, device="cuda", dtype=torch.int8) * 2 - 1).to(dt)
    pitch = _lib.lib.dbf_canonical_pitch_words(cols)
    words = torch.empty((rows, pitch), dtype=torch.int32, device="cuda")
    bad = torch.empty((), dtype=torch.int64, device="cuda")
    back = torch.empty_like(dense)
    for _ in range(2):
        _lib.check(_lib.lib.dbf_pack_signs(dense.data_ptr(), _lib.dtype_code(dt), rows, cols, cols, words.data_ptr(), pitch, bad.data_ptr(), _lib.stream_ptr()), "pack")
        _lib.check(_lib.lib.dbf_unpack_signs(words.data_ptr(), rows, cols, pitch, back.data_ptr(), _lib.dtype_code(dt), cols, _lib.stream_ptr()), "unpack")
torch.cuda.synchronize(); print("ok")
