timeout 600 python -m pytest tests/test_shist.py -q -x > gpurun_out/pytest_shist.log 2>&1; echo "shist tests rc=$?"; tail -5 gpurun_out/pytest_shist.log
timeout 300 python tools/time_shist.py c2 2>&1 | tail -4
