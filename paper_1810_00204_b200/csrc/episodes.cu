// episodes.cu — qvts_run_episodes.
#include "qvts_internal.cuh"

using namespace qvts;

extern "C" qvts_status qvts_run_episodes(qvts_model *m, const qvts_episode_cfg *cfg, const qvts_comm *comm,
                                         qvts_episode_record *out_host, void *stream) {
    (void)m; (void)cfg; (void)comm; (void)out_host; (void)stream;
    set_error("qvts_run_episodes: not built yet");
    return QVTS_ERR_STATE;
}
