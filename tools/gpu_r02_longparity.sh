#!/bin/bash
# long parity runs on the current library: 20,000 seeded fuzz cases + every element of C2-C5
O=${OUT:-gpurun_out/r02/longparity}; mkdir -p $O
python -c "import paper_1805_07339_b200 as s; print(s.scn_version())" > $O/library.txt
SCN_FUZZ_CASES=20000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider > $O/pytest_fuzz20000.log 2>&1; echo "fuzz rc=$?"; tail -1 $O/pytest_fuzz20000.log
SCN_EXHAUSTIVE=1 timeout 2400 python -m pytest tests/test_gpu_exhaustive.py -q -p no:cacheprovider --durations=0 > $O/pytest_gpu_exhaustive.log 2>&1; echo "exhaustive rc=$?"; tail -1 $O/pytest_gpu_exhaustive.log
