set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reference_suites.py tests/test_dropin_gpu.py -q -rA > gpurun_out/r2c_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_ref.log
(cd tests/cpp/_reftests && timeout 600 ./unit_tests > ../../../gpurun_out/r2c_unit.txt 2>&1; echo "rc=$?" >> ../../../gpurun_out/r2c_unit.txt; timeout 600 ./acceptance > ../../../gpurun_out/r2c_accept.txt 2>&1; echo "rc=$?" >> ../../../gpurun_out/r2c_accept.txt)
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2c_t.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_t.log
tail -3 gpurun_out/r2c_ref.log gpurun_out/r2c_t.log
