# GPU parity run: pytest -m gpu (+ smoke) into gpurun_out/$1
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-tests}; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/status
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf ${PYTEST_ARGS} > $O/pytest.log 2>&1; echo pytest=$? >> $O/status
