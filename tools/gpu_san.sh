cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
TAG=r2c ONLY=memcheck bash tools/sanitize.sh
TAG=r2c ONLY=synccheck bash tools/sanitize.sh
