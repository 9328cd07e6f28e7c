# run the bf16 parity tests against a library variant: bash tools/gpu/variant_test.sh NAME
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
cp tools/liboomb_$1.so paper_2602_02108_b200/liboomb.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "bf16 or tc_forward or properties or degenerates" 2>&1 | tail -3
cat > /tmp/err.py <<'PY'
import numpy as np, sys
sys.path.insert(0, ".")
from tests.test_gpu_parity import ATTN_CASES, attn_case, bf16_case, run_device, run_oracle, rel
for name in ("qwen_sparse", "qwen_partial", "c1_dense"):
    mk, past, seed, sel = ATTN_CASES[name]
    c = mk()
    case = bf16_case(attn_case(c, past, seed=seed, dtype=np.float32, selected=sel))
    got, _ = run_device(c, case, "bf16")
    want = run_oracle(c, case)
    print(name, {k: "%.2e" % rel(got[k], want[k]) for k in ("out", "lse", "dq", "dk_cur", "grad_k")})
PY
python /tmp/err.py 2>&1 | grep -v Warn | tail -3
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
python /tmp/err.py 2>&1 | grep -v Warn | tail -3
