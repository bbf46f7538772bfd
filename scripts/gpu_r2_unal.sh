# Round 2: K2t2 UNAL (uint8 rows at any byte offset through the TMA ring): parity + widths.
set -u
mkdir -p gpurun_out/un
timeout -k 10 900 python -m pytest tests/test_gpu_unal_tma.py -q -x -p no:cacheprovider > gpurun_out/un/pytest_unal.log 2>&1; echo "rc=$?" >> gpurun_out/un/pytest_unal.log
timeout -k 10 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py tests/test_gpu_strided.py tests/test_gpu_dropin.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/un/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/un/pytest.log
timeout -k 10 600 python scripts/u8_widths.py > gpurun_out/un/u8w.log 2>&1
BITEDGE_NO_TMA_UNAL=1 timeout -k 10 600 python scripts/u8_widths.py > gpurun_out/un/u8w_no.log 2>&1
echo done
