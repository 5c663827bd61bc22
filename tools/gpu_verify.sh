#!/bin/bash
# Final verification: GPU suite, smoke, C++ facade + reference-plugin programs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/verify
O=gpurun_out/verify
timeout 900 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 300 ./tests/cpp/facade_test gpu > $O/facade.txt 2>&1; echo "rc=$?" >> $O/facade.txt
timeout 300 ./tests/cpp/ref_plugin_test > $O/ref_plugin.txt 2>&1; echo "rc=$?" >> $O/ref_plugin.txt
