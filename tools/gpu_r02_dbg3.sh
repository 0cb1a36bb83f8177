make tuning > /dev/null 2>&1
SCN_TEST_VERBOSE=1 SCN_LIB=tuning SCN_GRID=7 timeout 60 python tests/helpers/variant_parity.py 2>&1 | tail -5
