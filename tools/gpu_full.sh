set -x
O=gpurun_out/r02y
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
tools/checked_run.sh $O
bash tools/profile_r02.sh > $O/profile.log 2>&1
