# the reference's own test suite (copied, unmodified, to the git-ignored
# baseline/_reftests in the build container) run against this repo's drop-in
# through the `csrk` alias, on a B200
mkdir -p gpurun_out
cd baseline/_reftests && PYTHONPATH=$GRAFT_REPO_ROOT timeout 1500 python -m pytest -q -p no:cacheprovider -c /dev/null --rootdir . . > ../../gpurun_out/reftests.log 2>&1; echo "rc=$?" >> ../../gpurun_out/reftests.log
tail -15 ../../gpurun_out/reftests.log
