#!/bin/bash
O=gpurun_out/r2_t67; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log; grep -E "^E " $O/pytest.log | head -5
