/* Links a plain C program against libgridadmm.so through the reference
 * header layout (#include <gridadmm/gridadmm.h>) and exercises the host-only
 * part of the ABI (proj/tests/test_capi.cpp:47-94 semantics). */
#include <stdio.h>
#include <string.h>

#include <gridadmm/gridadmm.h>

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    gridadmm_network* net = NULL;
    if (gridadmm_network_load(argv[1], &net) != GRIDADMM_OK) return 3;
    if (gridadmm_network_num_buses(net) != 9 || gridadmm_network_num_generators(net) != 3 ||
        gridadmm_network_num_branches(net) != 9) return 4;
    gridadmm_network* missing = NULL;
    if (gridadmm_network_load("/no/such/case.m", &missing) != GRIDADMM_ERR_PARSE) return 5;
    if (!strstr(gridadmm_last_error(), "/no/such/case.m")) return 6;
    gridadmm_config* cfg = gridadmm_config_new();
    double v = 0.0;
    if (gridadmm_config_preset(cfg, "case9") != GRIDADMM_OK) return 7;
    if (gridadmm_config_get(cfg, "rho_pq", &v) != GRIDADMM_OK || v != 100.0) return 8;
    if (gridadmm_config_set(cfg, "max_inner", 1.5) != GRIDADMM_ERR_INVALID_ARG) return 9;
    if (gridadmm_network_num_buses(NULL) != 0) return 10;
    gridadmm_network_free(NULL);
    gridadmm_report_free(NULL);
    gridadmm_track_free(NULL);
    gridadmm_config_free(cfg);
    gridadmm_network_free(net);
    puts("ok");
    return 0;
}
