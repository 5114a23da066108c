# phase profile of the strip kernel for each set of build defines given as args ("" = default)
cd $GRAFT_REPO_ROOT
for d in "$@"; do
PRNU_NVCC_DEFS="PRNU_STRIP_PROFILE $d" python paper_1909_04573_b200/_build.py --force > /dev/null 2>&1 || echo buildfail
echo "== [$d]"; python tools/strip_phases.py 2>&1 | tail -15
done
