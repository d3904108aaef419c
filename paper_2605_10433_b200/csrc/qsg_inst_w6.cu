#define QSG_W 6
#include "qsg_inst.cuh"
